# GEMM1-overlapped gather: parity, interleaved A/B, launch lists
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 600 python -m pytest tests/test_gpu_gather_fused.py -m gpu -q -x --timeout 300 2>&1 | tail -15 > gpurun_out/r3c_pytest_gather.log
if grep -q " passed" gpurun_out/r3c_pytest_gather.log && ! grep -q "failed" gpurun_out/r3c_pytest_gather.log; then
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared.py tests/test_gpu_swap_tail.py tests/test_gpu_tail_split.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 600 2>&1 | tail -8 > gpurun_out/r3c_pytest_more.log
timeout 900 python scripts/ab.py --env BO_GATHER_FUSED=0 --workloads mixtral_prefill:0.5,qwen3_30b_a3b_prefill:0.5,qwen15_moe_a27b_prefill:0.5,mixtral_prefill:0.0 --reps 6 > gpurun_out/r3c_ab_gather.json 2> gpurun_out/r3c_ab_gather.err
for arm in 1 0; do
REPS=3 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 BO_GATHER_FUSED=$arm > gpurun_out/r3c_ncu_c4_g$arm.csv 2> gpurun_out/r3c_ncu_c4_g$arm.err
done
fi
cat gpurun_out/r3c_pytest_gather.log | tail -5; tail -3 gpurun_out/r3c_pytest_more.log; tail -3 gpurun_out/r3c_ab_gather.err
python - <<'P'
import json
d=json.load(open("gpurun_out/r3c_ab_gather.json"))
for wl,v in d.items():
    if wl=="arms": continue
    for arm,r in v.items():
        print(wl,arm,r["ms_median"],r["kernel_ms"])
P
