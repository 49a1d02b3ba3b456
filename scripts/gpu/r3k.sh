# gather in the permute for wide permute grids (C2): parity, interleaved A/B, launch lists
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "gather_in_permute or engine_variants or fused_combine" 2>&1 | tail -5 > gpurun_out/r3k_pytest.log
if grep -q " passed" gpurun_out/r3k_pytest.log && ! grep -q "failed\|rror" gpurun_out/r3k_pytest.log; then
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x --timeout 600 2>&1 | tail -3 >> gpurun_out/r3k_pytest.log
timeout 900 python scripts/ab.py --env BO_PERMUTE_GATHER=0 --workloads mixtral_prefill:0.5,mixtral_prefill:0.0 --reps 8 > gpurun_out/r3k_ab_permute_gather.json 2> gpurun_out/r3k_ab_permute_gather.err
for arm in 1 0; do
  REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_prefill 0.5 BO_PERMUTE_GATHER=$arm > gpurun_out/r3k_launches_c2_pg$arm.csv 2> gpurun_out/r3k_launches_c2_pg$arm.err
  python scripts/launch_summary.py gpurun_out/r3k_launches_c2_pg$arm.csv > gpurun_out/r3k_launches_c2_pg${arm}_summary.json
done
fi
cat gpurun_out/r3k_pytest.log
python - <<'P'
import json
d=json.load(open("gpurun_out/r3k_ab_permute_gather.json"))
for wl,v in d.items():
    if wl=="arms": continue
    for arm,r in v.items():
        print(wl,arm,r["ms_median"],r["kernel_ms"])
P
for f in gpurun_out/r3k_launches_*_summary.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['step_us'], [(k['kernel'][:40], k['us']) for k in d['kernels']])"; done
