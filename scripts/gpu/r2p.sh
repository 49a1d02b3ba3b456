python -c "from paper_2507_17133_b200.build import build; build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared.py tests/test_gpu_api.py -m gpu -q -x --timeout 600 2>&1 | tail -4 > gpurun_out/r2p_pytest.log
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r2p_launches_c4.csv 2> gpurun_out/r2p_launches_c4.err
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py qwen15_moe_a27b_prefill 0.8 > gpurun_out/r2p_launches_f2.csv 2> gpurun_out/r2p_launches_f2.err
tail -3 gpurun_out/r2p_pytest.log
