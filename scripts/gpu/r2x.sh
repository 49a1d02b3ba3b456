# final round-2 measurement: full GPU suite, smoke, bench (default), headline launch list, sanitizer incl. tail split
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2x_smi.txt
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -15 > gpurun_out/r2x_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2x_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-sweep --no-extra --no-cpu > gpurun_out/r2x_launches_bench.csv 2> gpurun_out/r2x_launches_bench.err
mkdir -p gpurun_out/sanitizer_r02b
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_r02b/san_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitizer_r02b/san_$t.log
done
tail -2 gpurun_out/r2x_pytest_gpu.log; tail -1 gpurun_out/r2x_smoke.log; tail -c 300 gpurun_out/r2x_bench.json; for f in gpurun_out/sanitizer_r02b/*.log; do tail -2 $f; done
