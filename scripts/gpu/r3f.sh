# full ncu (source page) of the C4 tcgen05 router and the C3 ratio-1 fused decode routing
python -c "from paper_2507_17133_b200.build import build; build()"
REPS=2 python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r3f_plain_c4.log 2>&1 && \
REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm -c 1 -o gpurun_out/r3f_c4_router python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r3f_ncu_c4.log 2>&1
REPS=2 python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r3f_plain_c3.log 2>&1 && \
REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_fused -s 1 -c 1 -o gpurun_out/r3f_c3_route_fused python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r3f_ncu_c3.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -2 gpurun_out/r3f_ncu_c4.log gpurun_out/r3f_ncu_c3.log
