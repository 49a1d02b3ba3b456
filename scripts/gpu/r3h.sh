# final measurement set of the round: smoke, bench (default command, twice), headline launch list,
# full ncu of the C2 FFN GEMMs, reference arm, full GPU suite
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r3h_smi.txt
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3h_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r3h_bench.json 2> gpurun_out/r3h_bench.err
timeout 900 python bench.py --no-sweep --no-extra --no-cpu > gpurun_out/r3h_bench2.json 2> gpurun_out/r3h_bench2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-sweep --no-extra --no-cpu > gpurun_out/r3h_launches_bench.csv 2> gpurun_out/r3h_launches_bench.err
python scripts/launch_summary.py gpurun_out/r3h_launches_bench.csv > gpurun_out/r3h_launches_bench_summary.json
REPS=2 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_grouped_gemm" --launch-skip 3 --launch-count 2 -o gpurun_out/r3h_c2_gemms python scripts/ffn_ncu_ab.py mixtral_prefill 0.5 > gpurun_out/r3h_ncu_c2.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3h_bench_reference.json 2> gpurun_out/r3h_bench_reference.err
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -8 > gpurun_out/r3h_pytest_gpu.log
tail -1 gpurun_out/r3h_smoke.log; tail -3 gpurun_out/r3h_pytest_gpu.log
python -c "
import json
for f in ('gpurun_out/r3h_bench.json','gpurun_out/r3h_bench2.json'):
    d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])
"
python -c "import json; d=json.load(open('gpurun_out/r3h_launches_bench_summary.json')); print(d['step_us'], [(k['kernel'][:45], k['us'], k['share']) for k in d['kernels']])"
