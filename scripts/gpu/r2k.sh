python -c "from paper_2507_17133_b200.build import build; build()"
timeout 300 python scripts/debug_router_m32.py > gpurun_out/r2k_debug.log 2>&1
timeout 900 python -m pytest tests/test_gpu_router_exact.py tests/test_gpu_streamk.py -m gpu -q --timeout 300 2>&1 | tail -8 > gpurun_out/r2k_pytest.log
timeout 600 python scripts/ab.py --env BO_ROUTE_FUSED=0 --workloads mixtral_decode:1.0,mixtral_decode:0.0 --reps 6 > gpurun_out/r2k_ab_route_fused.json 2> gpurun_out/r2k_ab_route_fused.err
cat gpurun_out/r2k_debug.log; tail -3 gpurun_out/r2k_pytest.log; tail -2 gpurun_out/r2k_ab_route_fused.err
