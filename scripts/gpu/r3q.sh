# combine of split-K partials with every split's load in flight: tests, C3 launch lists
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_api.py -m gpu -q -x --timeout 600 2>&1 | tail -3 > gpurun_out/r3q_pytest.log
if grep -q " passed" gpurun_out/r3q_pytest.log && ! grep -q "failed\|rror" gpurun_out/r3q_pytest.log; then
for wl in mixtral_decode:1.0 mixtral_decode:0.5; do
  n=${wl%%:*}; r=${wl##*:}
  REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py $n $r > gpurun_out/r3q_launches_${n}_$r.csv 2> gpurun_out/r3q_launches_${n}_$r.err
  python scripts/launch_summary.py gpurun_out/r3q_launches_${n}_$r.csv > gpurun_out/r3q_launches_${n}_${r}_summary.json
done
fi
cat gpurun_out/r3q_pytest.log
for f in gpurun_out/r3q_launches_*_summary.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['step_us'], [(k['kernel'][:40], k['us']) for k in d['kernels']])"; done
