python -c "from paper_2507_17133_b200.build import build; build(); build(variant='probe')"
timeout 900 python -m pytest tests/test_gpu_decode_swap.py -m gpu -q -x --timeout 300 2>&1 | tail -30 > gpurun_out/r2o_pytest_dec.log
timeout 600 python scripts/ab.py --env BO_DECODE_SWAP=0 --workloads mixtral_decode:1.0,mixtral_decode:0.5,mixtral_decode:0.0 --reps 6 > gpurun_out/r2o_ab_dec.json 2> gpurun_out/r2o_ab_dec.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_decode 1.0 > gpurun_out/r2o_probe_c3r1.json 2> gpurun_out/r2o_probe.err
tail -5 gpurun_out/r2o_pytest_dec.log; tail -4 gpurun_out/r2o_ab_dec.err
