L=paper_2507_17133_b200
cp $L/libbrownout.so /tmp/new.so
for wl in ${WLS:-"qwen3_30b_a3b_prefill 0.5" "qwen15_moe_a27b_prefill 0.8" "mixtral_prefill 0.5"}; do
 for r in 1 2 3; do
  for arm in prev new; do
   if [ $arm = prev ]; then cp $L/libbrownout_prev.so.bak $L/libbrownout.so; else cp /tmp/new.so $L/libbrownout.so; fi
   ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_grouped_gemm --csv python scripts/ffn_ncu_ab.py $wl 2>/dev/null | grep k_grouped | sed "s/^/$arm|$wl|/" >> gpurun_out/libab.csv
  done
 done
done
cp /tmp/new.so $L/libbrownout.so
python3 - <<'PY'
import csv, statistics, collections
by = collections.defaultdict(list)
for line in open("gpurun_out/libab.csv"):
    arm, wl, rest = line.split("|", 2)
    r = next(csv.reader([rest]))
    name = next(c for c in r if "k_grouped_gemm" in c)
    t = name.split("<", 1)[1].split(">")[0].replace("__nv_bfloat16, ", "").replace(" ", "")
    by[(wl, t, arm)].append(float(r[-1].replace(",", "")))
for k in sorted(by):
    print(k, round(statistics.median(by[k]) / 1e3, 1), len(by[k]))
PY
