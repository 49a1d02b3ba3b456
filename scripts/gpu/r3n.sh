# extended parity soak on the final code + full GPU suite at HEAD
python -c "from paper_2507_17133_b200.build import build; build()"
mkdir -p gpurun_out/soak_r02b
timeout 2400 python scripts/soak.py --n 2000 --seed 23 > gpurun_out/soak_r02b/soak_2000_seed23.log 2>&1; echo "soak rc=$?" >> gpurun_out/soak_r02b/soak_2000_seed23.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -6 > gpurun_out/r3n_pytest_gpu.log
tail -3 gpurun_out/soak_r02b/soak_2000_seed23.log; tail -3 gpurun_out/r3n_pytest_gpu.log
