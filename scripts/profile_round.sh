set -x
python bench.py > gpurun_out/r01c_bench_final.json 2> gpurun_out/r01c_bench_final.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r01c_launches_bench.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1
REPS=1 ncu --set full --clock-control none --import-source on -k regex:k_grouped_gemm -c 2 --csv --page raw --log-file gpurun_out/r01c_c2_ffn_gemms_ncu_raw.csv python scripts/ffn_ncu_ab.py mixtral_prefill 0.5 > /dev/null 2>&1
ls -la gpurun_out/r01c*
