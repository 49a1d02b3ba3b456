# bulk-copy gather / combine: parity, interleaved A/B, ncu DRAM bytes of both arms
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 900 python -m pytest tests/test_gpu_bulk_stream.py tests/test_gpu_parity.py tests/test_gpu_shared.py -m gpu -q -x --timeout 600 2>&1 | tail -15 > gpurun_out/r3a_pytest.log
timeout 900 python scripts/ab.py --env BO_BULK_STREAM=0 --workloads qwen3_30b_a3b_prefill:0.5,mixtral_prefill:0.5,qwen15_moe_a27b_prefill:0.5,mixtral_decode:0.0 --reps 6 > gpurun_out/r3a_ab_bulk.json 2> gpurun_out/r3a_ab_bulk.err
for arm in 1 0; do
REPS=3 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"gather|combine" --clock-control none --csv python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 BO_BULK_STREAM=$arm > gpurun_out/r3a_ncu_c4_bulk$arm.csv 2> gpurun_out/r3a_ncu_c4_bulk$arm.err
REPS=3 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"gather|combine" --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_prefill 0.5 BO_BULK_STREAM=$arm > gpurun_out/r3a_ncu_c2_bulk$arm.csv 2> gpurun_out/r3a_ncu_c2_bulk$arm.err
done
cat gpurun_out/r3a_pytest.log | tail -4; tail -3 gpurun_out/r3a_ab_bulk.err
python - <<'P'
import json
d=json.load(open("gpurun_out/r3a_ab_bulk.json"))
for wl,v in d.items():
    if wl=="arms": continue
    for arm,r in v.items():
        print(wl,arm,r["ms_median"],r["kernel_ms"])
P
