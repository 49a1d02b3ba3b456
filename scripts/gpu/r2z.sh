python -c "from paper_2507_17133_b200.build import build; build(); build(variant='probe')"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_swap_tail.py tests/test_gpu_fullsize.py -m gpu -q -x --timeout 600 2>&1 | tail -5 > gpurun_out/r2z_pytest.log
timeout 600 python scripts/ab.py --env BO_SWAP_TAIL=0 --workloads mixtral_decode:1.0,mixtral_decode:0.75 --reps 8 > gpurun_out/r2z_ab_swap2.json 2> gpurun_out/r2z_ab_swap2.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_decode 1.0 > gpurun_out/r2z_probe_c3r1.json 2> gpurun_out/r2z_probe.err
tail -3 gpurun_out/r2z_pytest.log; tail -3 gpurun_out/r2z_ab_swap2.err
