python -c "from paper_2507_17133_b200.build import build; build()"
timeout 1200 python -m pytest tests/test_gpu_router_exact.py tests/test_gpu_parity.py tests/test_gpu_shared.py tests/test_ep.py -m gpu -q -x --timeout 600 2>&1 | tail -4 > gpurun_out/r2v_pytest.log
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2v_launches_c3r1.csv 2> gpurun_out/r2v_launches_c3r1.err
BO_ROUTE_FUSED=0 REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2v_launches_c3r1_unfused.csv 2>> gpurun_out/r2v_launches_c3r1.err
timeout 600 python scripts/ab.py --env BO_ROUTE_FUSED=0 --workloads mixtral_decode:1.0,mixtral_decode:0.0 --reps 8 > gpurun_out/r2v_ab_route_fused.json 2> gpurun_out/r2v_ab_route_fused.err
tail -3 gpurun_out/r2v_pytest.log; tail -3 gpurun_out/r2v_ab_route_fused.err
