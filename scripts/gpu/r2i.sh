# fused decode routing v2 (warp-synchronous Alg. 1), router top-K insertion, NCCL test in a child
python -c "from paper_2507_17133_b200.build import build; build(); build(variant='probe')"
timeout 1200 python -m pytest tests/test_gpu_router_exact.py tests/test_ep.py tests/test_gpu_shared.py tests/test_gpu_api.py -m gpu -q -x --timeout 600 2>&1 | tail -15 > gpurun_out/r2i_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1
timeout 600 python scripts/ab.py --env BO_ROUTE_FUSED=0 --workloads mixtral_decode:1.0,mixtral_decode:0.0,qwen3_30b_a3b_prefill:0.5 --reps 6 > gpurun_out/r2i_ab_route_fused.json 2> gpurun_out/r2i_ab_route_fused.err
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2i_launches_c3r1.csv 2> gpurun_out/r2i_launches_c3r1.err
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r2i_launches_c4.csv 2> gpurun_out/r2i_launches_c4.err
cat gpurun_out/r2i_pytest.log | tail -3; cat gpurun_out/r2i_smoke.log | tail -2; cat gpurun_out/r2i_ab_route_fused.err | tail -3
