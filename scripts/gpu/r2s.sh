# final-ish measurement set: bench (default command), launch list of the headline bench command, full ncu of C2 FFN GEMMs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2s_smi.txt
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 900 python bench.py > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-sweep --no-extra --no-cpu > gpurun_out/r2s_launches_bench.csv 2> gpurun_out/r2s_launches_bench.err
REPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_grouped_gemm" --launch-skip 3 --launch-count 2 -o gpurun_out/r2s_c2_gemms python scripts/ffn_ncu_ab.py mixtral_prefill 0.5 > gpurun_out/r2s_ncu_c2.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2s_bench_reference.json 2> gpurun_out/r2s_bench_reference.err
tail -c 400 gpurun_out/r2s_bench.json; tail -2 gpurun_out/r2s_ncu_c2.log
