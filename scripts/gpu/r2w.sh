python -c "from paper_2507_17133_b200.build import build; build(); build(variant='probe')"
timeout 900 python -m pytest tests/test_gpu_tail_split.py tests/test_gpu_parity.py tests/test_gpu_shared.py tests/test_c_client.py -m gpu -q -x --timeout 300 2>&1 | tail -8 > gpurun_out/r2w_pytest.log
timeout 900 python scripts/ab.py --env BO_TAIL_SPLIT=0 --workloads mixtral_prefill:0.5,mixtral_prefill:0.0,mixtral_prefill:1.0 --reps 8 > gpurun_out/r2w_ab_tail_split.json 2> gpurun_out/r2w_ab_tail_split.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_prefill 0.5 > gpurun_out/r2w_probe_c2.json 2> gpurun_out/r2w_probe.err
tail -3 gpurun_out/r2w_pytest.log; tail -3 gpurun_out/r2w_ab_tail_split.err
