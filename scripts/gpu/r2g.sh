# NCCL diagnosis (the world-1 library NCCL test hung in r2f), decode GEMM1 schedule A/B, full ncu captures
python -c "from paper_2507_17133_b200.build import build; build()"
ip -o addr 2>/dev/null | head -5 > gpurun_out/r2g_net.log; ls /sys/class/net >> gpurun_out/r2g_net.log
NCCL_DEBUG=INFO timeout 120 python scripts/nccl_torch_probe.py > gpurun_out/r2g_nccl_torch.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_nccl_torch.log
NCCL_DEBUG=INFO timeout 120 python scripts/nccl_probe.py 0 > gpurun_out/r2g_nccl_lib_exact.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_nccl_lib_exact.log
NCCL_DEBUG=INFO timeout 120 python scripts/nccl_probe.py 1 > gpurun_out/r2g_nccl_lib_padded.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_nccl_lib_padded.log
NCCL_DEBUG=INFO NCCL_SOCKET_IFNAME=lo timeout 120 python scripts/nccl_probe.py 1 > gpurun_out/r2g_nccl_lib_padded_lo.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_nccl_lib_padded_lo.log
timeout 900 python scripts/ab.py --env BO_PAIR_ROWS1=256 --env "BO_PAIR_ROWS1=256;BO_SWAP_TAIL=0" --env BO_B_POLICY=0 --env BO_TILE_ALT=0 --workloads mixtral_decode:1.0,mixtral_decode:0.5 --reps 6 > gpurun_out/r2g_ab_decode.json 2> gpurun_out/r2g_ab_decode.err
REPS=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_grouped_gemm" --launch-skip 3 --launch-count 3 -o gpurun_out/r2g_c4 python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r2g_ncu_c4.log 2>&1
REPS=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_grouped_gemm" --launch-skip 2 --launch-count 2 -o gpurun_out/r2g_c3r1 python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2g_ncu_c3r1.log 2>&1
REPS=2 BO_PAIR_ROWS1=256 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_grouped_gemm" --launch-skip 2 --launch-count 2 -o gpurun_out/r2g_c3r1_pair python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2g_ncu_c3r1_pair.log 2>&1
tail -3 gpurun_out/r2g_nccl_*.log; cat gpurun_out/r2g_ab_decode.err | tail -5
