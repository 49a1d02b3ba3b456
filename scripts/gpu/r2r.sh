python -c "from paper_2507_17133_b200.build import build; build(); build(variant='probe')"
timeout 900 python -m pytest tests/test_gpu_half_tail.py tests/test_gpu_parity.py -m gpu -q -x --timeout 300 2>&1 | tail -5 > gpurun_out/r2r_pytest.log
timeout 900 python scripts/ab.py --env BO_HALF_TAIL=0 --workloads mixtral_prefill:0.5,mixtral_prefill:0.0,mixtral_prefill:0.25,qwen3_30b_a3b_prefill:0.5 --reps 6 > gpurun_out/r2r_ab_half_tail.json 2> gpurun_out/r2r_ab_half_tail.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_prefill 0.5 > gpurun_out/r2r_probe_c2.json 2> gpurun_out/r2r_probe.err
tail -3 gpurun_out/r2r_pytest.log; tail -5 gpurun_out/r2r_ab_half_tail.err
