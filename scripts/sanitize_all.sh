mkdir -p gpurun_out/sanitizer_r01c
python scripts/sanitize_run.py > gpurun_out/sanitizer_r01c/san_plain.log 2>&1; tail -2 gpurun_out/sanitizer_r01c/san_plain.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_r01c/san_$t.log 2>&1
  echo "$t rc=$?"; tail -2 gpurun_out/sanitizer_r01c/san_$t.log
done
# initcheck does not see bytes written by TMA bulk stores (async proxy): GEMM2's Yp slabs
# read by k_combine show as uninitialised.  The same run with plain stores must be clean.
BO_TMA_STORE=0 timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_r01c/san_initcheck_plain_stores.log 2>&1
echo "initcheck (BO_TMA_STORE=0) rc=$?"; tail -2 gpurun_out/sanitizer_r01c/san_initcheck_plain_stores.log
