# atomics-free histograms: parity; decode GEMM1 pairs A/B; launch lists + full captures (C4 GEMM2, C4 router, C3 r1 GEMM1)
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 900 python -m pytest tests/test_gpu_router_exact.py tests/test_gpu_parity.py -m gpu -q -x --timeout 300 2>&1 | tail -15 > gpurun_out/r2d_pytest.log
timeout 600 python scripts/ab.py --env BO_PAIR_ROWS1=256 --env "BO_PAIR_ROWS1=256;BO_SWAP_TAIL=0" --workloads mixtral_decode:1.0,mixtral_decode:0.5 --reps 6 > gpurun_out/r2d_ab_decode_pairs.json 2> gpurun_out/r2d_ab_decode_pairs.err
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r2d_launches_c4.csv 2> gpurun_out/r2d_launches_c4.err
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2d_launches_c3r1.csv 2> gpurun_out/r2d_launches_c3r1.err
REPS=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_grouped_gemm" --launch-skip 4 --launch-count 3 -o gpurun_out/r2d_c4_gemms python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r2d_ncu_c4.log 2>&1
REPS=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_grouped_gemm" --launch-skip 4 --launch-count 3 -o gpurun_out/r2d_c3r1_gemms python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2d_ncu_c3r1.log 2>&1
tail -3 gpurun_out/r2d_pytest.log; cat gpurun_out/r2d_ab_decode_pairs.err
