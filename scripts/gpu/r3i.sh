# parity soak on the round's final code (random shapes / ratios / modes / knobs vs the fp64 oracle)
python -c "from paper_2507_17133_b200.build import build; build()"
mkdir -p gpurun_out/soak_r02b
timeout 1500 python scripts/soak.py --n 400 --seed 11 > gpurun_out/soak_r02b/soak_400_seed11.log 2>&1; echo "soak rc=$?" >> gpurun_out/soak_r02b/soak_400_seed11.log
tail -3 gpurun_out/soak_r02b/soak_400_seed11.log
