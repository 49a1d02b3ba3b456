# router two-list top-K + NVTX ranges: router tests, C4 / f2 launch lists, full GPU suite, smoke, bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r3g_smi.txt
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 600 python -m pytest tests/test_gpu_router_exact.py -m gpu -q -x --timeout 300 2>&1 | tail -5 > gpurun_out/r3g_pytest_router.log
for wl in qwen3_30b_a3b_prefill:0.5 qwen15_moe_a27b_prefill:0.5; do
  n=${wl%%:*}; r=${wl##*:}
  REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py $n $r > gpurun_out/r3g_launches_$n.csv 2> gpurun_out/r3g_launches_$n.err
  python scripts/launch_summary.py gpurun_out/r3g_launches_$n.csv > gpurun_out/r3g_launches_${n}_summary.json
done
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -8 > gpurun_out/r3g_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3g_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r3g_bench.json 2> gpurun_out/r3g_bench.err
tail -2 gpurun_out/r3g_pytest_router.log; tail -3 gpurun_out/r3g_pytest_gpu.log; tail -1 gpurun_out/r3g_smoke.log
for f in gpurun_out/r3g_launches_*_summary.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['step_us'], [(k['kernel'][:45], k['us']) for k in d['kernels']])"; done
python -c "import json; d=json.load(open('gpurun_out/r3g_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
