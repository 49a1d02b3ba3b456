# serpentine k-order: parity with BO_SERPENTINE=3, interleaved A/B, ncu DRAM bytes
python -c "from paper_2507_17133_b200.build import build; build()"
BO_SERPENTINE=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tail_split.py tests/test_gpu_swap_tail.py -m gpu -q -x --timeout 600 2>&1 | tail -4 > gpurun_out/r3m_pytest.log
if grep -q " passed" gpurun_out/r3m_pytest.log && ! grep -q "failed\|rror" gpurun_out/r3m_pytest.log; then
timeout 1200 python scripts/ab.py --env BO_SERPENTINE=1 --env BO_SERPENTINE=2 --env BO_SERPENTINE=3 --workloads mixtral_prefill:0.5,qwen3_30b_a3b_prefill:0.5,mixtral_decode:0.0,mixtral_decode:1.0 --reps 6 > gpurun_out/r3m_ab_serp.json 2> gpurun_out/r3m_ab_serp.err
for arm in 0 3; do
REPS=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:k_grouped_gemm --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_prefill 0.5 BO_SERPENTINE=$arm > gpurun_out/r3m_ncu_c2_s$arm.csv 2> gpurun_out/r3m_ncu_c2_s$arm.err
REPS=2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:k_grouped_gemm --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_decode 0.0 BO_SERPENTINE=$arm > gpurun_out/r3m_ncu_c3_s$arm.csv 2> gpurun_out/r3m_ncu_c3_s$arm.err
done
fi
cat gpurun_out/r3m_pytest.log
python - <<'P'
import json
d=json.load(open("gpurun_out/r3m_ab_serp.json"))
for wl,v in d.items():
    if wl=="arms": continue
    for arm,r in v.items():
        print(wl,arm,r["ms_median"],{k:round(x*1000,1) for k,x in r["kernel_ms"].items() if 'gemm' in k})
P
for f in gpurun_out/r3m_ncu_*.csv; do echo $f; grep -E "dram__bytes_read.sum|gpu__time_duration|lts__t_sector_hit" $f | awk -F'","' '{print substr($5,1,45), $(NF-2), $NF}' | tail -6; done
