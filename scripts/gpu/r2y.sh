python -c "from paper_2507_17133_b200.build import build; build()"
mkdir -p gpurun_out/sanitizer_r02c
for t in racecheck memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_r02c/san_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitizer_r02c/san_$t.log
done
BO_TMA_STORE=0 timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_r02c/san_initcheck_plain_stores.log 2>&1; echo "initcheck rc=$?" >> gpurun_out/sanitizer_r02c/san_initcheck_plain_stores.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -8 > gpurun_out/r2y_pytest_gpu.log
for f in gpurun_out/sanitizer_r02c/*.log; do echo $f; tail -2 $f; done; tail -2 gpurun_out/r2y_pytest_gpu.log
