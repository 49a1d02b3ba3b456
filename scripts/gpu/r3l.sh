# L2 policy of the weight tiles at prefill (C2): interleaved A/B and ncu DRAM bytes of both GEMMs
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 900 python scripts/ab.py --env BO_B_POLICY=1 --workloads mixtral_prefill:0.5 --reps 8 > gpurun_out/r3l_ab_bpolicy.json 2> gpurun_out/r3l_ab_bpolicy.err
for arm in 0 1; do
REPS=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:k_grouped_gemm --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_prefill 0.5 BO_B_POLICY=$arm > gpurun_out/r3l_ncu_c2_bp$arm.csv 2> gpurun_out/r3l_ncu_c2_bp$arm.err
done
python - <<'P'
import json
d=json.load(open("gpurun_out/r3l_ab_bpolicy.json"))
for wl,v in d.items():
    if wl=="arms": continue
    for arm,r in v.items():
        print(wl,arm,r["ms_median"],r["kernel_ms"])
P
for arm in 0 1; do echo arm $arm; grep -E "dram__bytes_read.sum|gpu__time_duration|lts__t_sector_hit" gpurun_out/r3l_ncu_c2_bp$arm.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | tail -8; done
