# decode routing: x rows leave the fused routing kernel by TMA bulk stores; tests, launch lists, probe
python -c "from paper_2507_17133_b200.build import build; build()"
python -m paper_2507_17133_b200.build --variant probe > /dev/null
timeout 900 python -m pytest tests/test_gpu_router_exact.py tests/test_gpu_parity.py tests/test_gpu_shared.py tests/test_gpu_api.py -m gpu -q -x --timeout 600 2>&1 | tail -4 > gpurun_out/r3p_pytest.log
if grep -q " passed" gpurun_out/r3p_pytest.log && ! grep -q "failed\|rror" gpurun_out/r3p_pytest.log; then
for wl in mixtral_decode:1.0 mixtral_decode:0.0 tiny:0.5; do
  n=${wl%%:*}; r=${wl##*:}
  REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py $n $r > gpurun_out/r3p_launches_${n}_$r.csv 2> gpurun_out/r3p_launches_${n}_$r.err
  python scripts/launch_summary.py gpurun_out/r3p_launches_${n}_$r.csv > gpurun_out/r3p_launches_${n}_${r}_summary.json
  BO_LIB=probe timeout 300 python scripts/probe_route.py $n $r > gpurun_out/r3p_probe_route_${n}_$r.json 2> gpurun_out/r3p_probe_route_${n}_$r.err
done

fi
cat gpurun_out/r3p_pytest.log
for f in gpurun_out/r3p_launches_*_summary.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['step_us'], [(k['kernel'][:40], k['us']) for k in d['kernels']])"; done
for f in gpurun_out/r3p_probe_route_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); [print(r['ctas'], r['phase_median_ns']) for r in d['runs'][:3]]"; done
python - <<'P'
import json
for wl,v in d.items():
    if wl=="arms": continue
    for arm,r in v.items():
        print(wl,arm,r["ms_median"],{k:round(x*1000,1) for k,x in r["kernel_ms"].items()})
P
