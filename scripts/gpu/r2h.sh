# fused decode routing (parity + timing), NCCL world-1 test in a child process, per-tile probes
python -c "from paper_2507_17133_b200.build import build; build(); build(variant='probe')"
timeout 900 python -m pytest tests/test_gpu_router_exact.py tests/test_ep.py -m gpu -q -x --timeout 600 2>&1 | tail -15 > gpurun_out/r2h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1
timeout 600 python scripts/ab.py --env BO_ROUTE_FUSED=0 --workloads mixtral_decode:1.0,mixtral_decode:0.0 --reps 6 > gpurun_out/r2h_ab_route_fused.json 2> gpurun_out/r2h_ab_route_fused.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_decode 1.0 > gpurun_out/r2h_probe_c3r1.json 2> gpurun_out/r2h_probe_c3r1.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_decode 1.0 BO_PAIR_ROWS1=256 > gpurun_out/r2h_probe_c3r1_pair.json 2>> gpurun_out/r2h_probe_c3r1.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_decode 0.5 > gpurun_out/r2h_probe_c3r05.json 2>> gpurun_out/r2h_probe_c3r1.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r2h_probe_c4.json 2>> gpurun_out/r2h_probe_c3r1.err
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2h_launches_c3r1.csv 2> gpurun_out/r2h_launches_c3r1.err
cat gpurun_out/r2h_pytest.log | tail -3; cat gpurun_out/r2h_smoke.log | tail -2; cat gpurun_out/r2h_ab_route_fused.err | tail -3; tail -2 gpurun_out/r2h_probe_c3r1.err
