# round-2 re-entry: full GPU suite + bench at HEAD, C3 r1 / C4 launch lists
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -40 > gpurun_out/r2f_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r2f_launches_c4.csv 2> gpurun_out/r2f_launches_c4.err
REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2f_launches_c3r1.csv 2> gpurun_out/r2f_launches_c3r1.err
tail -3 gpurun_out/r2f_pytest_gpu.log
