# tcgen05 router on expert-split CTA pairs (DSMEM merge of the top-K lists): exact tests, parity, A/B, launch lists
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 900 python -m pytest tests/test_gpu_router_exact.py -m gpu -q -x --timeout 600 2>&1 | tail -8 > gpurun_out/r3j_pytest_router.log
if grep -q " passed" gpurun_out/r3j_pytest_router.log && ! grep -q "failed\|rror" gpurun_out/r3j_pytest_router.log; then
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 600 2>&1 | tail -5 > gpurun_out/r3j_pytest_more.log
timeout 900 python scripts/ab.py --env BO_ROUTER_PAIR=0 --workloads qwen3_30b_a3b_prefill:0.5,qwen15_moe_a27b_prefill:0.5 --reps 8 > gpurun_out/r3j_ab_router_pair.json 2> gpurun_out/r3j_ab_router_pair.err
for arm in 1 0; do
  REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 BO_ROUTER_PAIR=$arm > gpurun_out/r3j_launches_c4_p$arm.csv 2> gpurun_out/r3j_launches_c4_p$arm.err
  python scripts/launch_summary.py gpurun_out/r3j_launches_c4_p$arm.csv > gpurun_out/r3j_launches_c4_p${arm}_summary.json
  REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py qwen15_moe_a27b_prefill 0.5 BO_ROUTER_PAIR=$arm > gpurun_out/r3j_launches_f2_p$arm.csv 2> gpurun_out/r3j_launches_f2_p$arm.err
  python scripts/launch_summary.py gpurun_out/r3j_launches_f2_p$arm.csv > gpurun_out/r3j_launches_f2_p${arm}_summary.json
done
fi
cat gpurun_out/r3j_pytest_router.log | tail -3; tail -2 gpurun_out/r3j_pytest_more.log
python - <<'P'
import json
d=json.load(open("gpurun_out/r3j_ab_router_pair.json"))
for wl,v in d.items():
    if wl=="arms": continue
    for arm,r in v.items():
        print(wl,arm,r["ms_median"],r["kernel_ms"])
P
for f in gpurun_out/r3j_launches_*_summary.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['step_us'], [(k['kernel'][:50], k['us']) for k in d['kernels']][:2])"; done
