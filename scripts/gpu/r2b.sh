# full GPU suite on the pruned engine + bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/r2b_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
tail -3 gpurun_out/r2b_pytest_gpu.log
