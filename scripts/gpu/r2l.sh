# full GPU suite after the fused-routing / NCCL-teardown changes; route_fused A/B; bench
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -30 > gpurun_out/r2l_pytest_gpu.log
timeout 600 python scripts/ab.py --env BO_ROUTE_FUSED=0 --workloads mixtral_decode:1.0,mixtral_decode:0.5,mixtral_decode:0.0 --reps 8 > gpurun_out/r2l_ab_route_fused.json 2> gpurun_out/r2l_ab_route_fused.err
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2l_launches_c3r1.csv 2> gpurun_out/r2l_launches_c3r1.err
tail -3 gpurun_out/r2l_pytest_gpu.log; tail -3 gpurun_out/r2l_ab_route_fused.err
