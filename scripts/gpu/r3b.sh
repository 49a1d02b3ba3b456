# session-3 start: state check after the container re-creation
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r3b_smi.txt
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3b_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r3b_bench.json 2> gpurun_out/r3b_bench.err
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -15 > gpurun_out/r3b_pytest_gpu.log
tail -1 gpurun_out/r3b_smoke.log; tail -c 600 gpurun_out/r3b_bench.json; tail -3 gpurun_out/r3b_pytest_gpu.log
