# robustness: parity soak (incl. the production router / fused routing), compute-sanitizer, full GPU suite
python -c "from paper_2507_17133_b200.build import build; build()"
mkdir -p gpurun_out/soak_r02 gpurun_out/sanitizer_r02
timeout 1800 python scripts/soak.py --n 500 --seed 7 > gpurun_out/soak_r02/soak_500_seed7.log 2>&1; echo "soak rc=$?" >> gpurun_out/soak_r02/soak_500_seed7.log
python scripts/sanitize_run.py > gpurun_out/sanitizer_r02/san_plain.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_r02/san_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitizer_r02/san_$t.log
done
BO_TMA_STORE=0 timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_r02/san_initcheck_plain_stores.log 2>&1; echo "initcheck rc=$?" >> gpurun_out/sanitizer_r02/san_initcheck_plain_stores.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -15 > gpurun_out/r2q_pytest_gpu.log
tail -2 gpurun_out/soak_r02/soak_500_seed7.log; for f in gpurun_out/sanitizer_r02/*.log; do echo $f; tail -2 $f; done; tail -2 gpurun_out/r2q_pytest_gpu.log
