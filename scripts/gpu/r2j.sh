# debug: router-exact stats on the tcgen05 path; stream-K parity + A/B
python -c "from paper_2507_17133_b200.build import build; build(); build(variant='probe')"
timeout 600 python -m pytest "tests/test_gpu_router_exact.py::test_every_router_exact_routing_and_output" -m gpu -q --timeout 300 -k "m32_tc" 2>&1 | tail -40 > gpurun_out/r2j_router_m32.log
timeout 900 python -m pytest tests/test_gpu_streamk.py -m gpu -q -x --timeout 300 2>&1 | tail -30 > gpurun_out/r2j_streamk.log
timeout 600 python scripts/ab.py --env BO_DECODE_STREAMK=0 --workloads mixtral_decode:1.0,mixtral_decode:0.5,mixtral_decode:0.0 --reps 6 > gpurun_out/r2j_ab_streamk.json 2> gpurun_out/r2j_ab_streamk.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_decode 1.0 > gpurun_out/r2j_probe_c3r1.json 2> gpurun_out/r2j_probe.err
tail -3 gpurun_out/r2j_router_m32.log; tail -3 gpurun_out/r2j_streamk.log; tail -4 gpurun_out/r2j_ab_streamk.err
