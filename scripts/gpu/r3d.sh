# router top-8 sorting network: exact-router tests, C4 / f2 launch lists; route_fused phase probe
python -c "from paper_2507_17133_b200.build import build; build()"
python -m paper_2507_17133_b200.build --variant probe > /dev/null
timeout 900 python -m pytest tests/test_gpu_router_exact.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 2>&1 | tail -8 > gpurun_out/r3d_pytest_router.log
for wl in qwen3_30b_a3b_prefill:0.5 qwen15_moe_a27b_prefill:0.5 mixtral_decode:1.0; do
  n=${wl%%:*}; r=${wl##*:}
  REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py $n $r > gpurun_out/r3d_launches_$n.csv 2> gpurun_out/r3d_launches_$n.err
  python scripts/launch_summary.py gpurun_out/r3d_launches_$n.csv > gpurun_out/r3d_launches_${n}_summary.json
done
for wl in mixtral_decode:1.0 mixtral_decode:0.0 tiny:0.5; do
  n=${wl%%:*}; r=${wl##*:}
  BO_LIB=probe timeout 300 python scripts/probe_route.py $n $r > gpurun_out/r3d_probe_route_${n}_$r.json 2> gpurun_out/r3d_probe_route_${n}_$r.err
done
tail -3 gpurun_out/r3d_pytest_router.log
for f in gpurun_out/r3d_launches_*_summary.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['step_us'], [(k['kernel'][:45], k['us']) for k in d['kernels']])"; done
for f in gpurun_out/r3d_probe_route_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); [print(r['ctas'], r['phase_median_ns'], r['phase_max_ns']) for r in d['runs']]"; done
