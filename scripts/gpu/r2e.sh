python -c "from paper_2507_17133_b200.build import build; build()"
ip -o addr 2>/dev/null | head; ls /sys/class/net
NCCL_DEBUG=INFO timeout 90 python scripts/nccl_probe.py 1 > gpurun_out/r2e_nccl_default.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_nccl_default.log
NCCL_DEBUG=INFO NCCL_SOCKET_IFNAME=lo timeout 90 python scripts/nccl_probe.py 1 > gpurun_out/r2e_nccl_lo.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_nccl_lo.log
NCCL_DEBUG=INFO NCCL_SOCKET_IFNAME=lo timeout 90 python scripts/nccl_probe.py 0 > gpurun_out/r2e_nccl_lo_exact.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_nccl_lo_exact.log
timeout 600 python -m pytest tests/test_c_client.py tests/test_gpu_api.py -m gpu -q -x --timeout 200 2>&1 | tail -15 > gpurun_out/r2e_pytest_api.log
bash scripts/gpu/r2d.sh
