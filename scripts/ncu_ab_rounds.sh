# Interleaved rounds of kernel-time A/B under ncu launch lists:
#   bash scripts/ncu_ab_rounds.sh ROUNDS "<workload> <ratio>" ENV1 ENV2 ...  ("-" = defaults)
# prints per arm and per grouped-GEMM instantiation the median duration over all
# rounds (scripts/ffn_ncu_ab.py runs 6 forwards per round).
rounds=$1; shift; wl=$1; shift
tmp=$(mktemp -d)
for r in $(seq 1 $rounds); do
  for e in "$@"; do
    f=$tmp/$(echo "$e" | tr '=;/ ' '____')
    ee=$e; if [ "$ee" = "-" ]; then ee=""; fi
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_grouped_gemm --csv python scripts/ffn_ncu_ab.py $wl $ee 2>/dev/null | grep k_grouped >> $f
  done
done
for e in "$@"; do
  f=$tmp/$(echo "$e" | tr '=;/ ' '____')
  python3 - "$f" "$wl" "$e" <<'PY'
import csv, sys, statistics
by = {}
for r in csv.reader(open(sys.argv[1])):
    name = next(c for c in r if "k_grouped_gemm" in c)
    tmpl = name.split("<", 1)[1].split(">")[0].replace("__nv_bfloat16, ", "").replace(" ", "")
    by.setdefault(tmpl, []).append(float(r[-1].replace(",", "")))
print(sys.argv[2], f"{sys.argv[3]:>20s}", "  ".join(f"<{k}> {statistics.median(v)/1e3:8.1f} us (n={len(v)})" for k, v in by.items()))
PY
done
