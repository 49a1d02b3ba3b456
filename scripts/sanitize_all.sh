mkdir -p gpurun_out/sanitizer_r01c
python scripts/sanitize_run.py > gpurun_out/sanitizer_r01c/san_plain.log 2>&1; tail -2 gpurun_out/sanitizer_r01c/san_plain.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_r01c/san_$t.log 2>&1
  echo "$t rc=$?"; tail -2 gpurun_out/sanitizer_r01c/san_$t.log
done
