set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 900 python -m pytest tests/test_gpu_router_exact.py -x -q 2>&1 | tail -30 > gpurun_out/r2a_router_exact.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q 2>&1 | tail -30 > gpurun_out/r2a_fullsize.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -30 > gpurun_out/r2a_parity.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
tail -5 gpurun_out/*.log
