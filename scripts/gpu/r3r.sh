# final validation at HEAD (TMA-bulk decode routing): full GPU suite, soak, smoke, bench, decode launch lists
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r3r_smi.txt
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -6 > gpurun_out/r3r_pytest_gpu.log
mkdir -p gpurun_out/soak_r02c
timeout 1800 python scripts/soak.py --n 1000 --seed 31 > gpurun_out/soak_r02c/soak_1000_seed31.log 2>&1; echo "soak rc=$?" >> gpurun_out/soak_r02c/soak_1000_seed31.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3r_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r3r_bench.json 2> gpurun_out/r3r_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-sweep --no-extra --no-cpu > gpurun_out/r3r_launches_bench.csv 2> gpurun_out/r3r_launches_bench.err
python scripts/launch_summary.py gpurun_out/r3r_launches_bench.csv > gpurun_out/r3r_launches_bench_summary.json
tail -3 gpurun_out/r3r_pytest_gpu.log; tail -2 gpurun_out/soak_r02c/soak_1000_seed31.log; tail -1 gpurun_out/r3r_smoke.log
python -c "
import json
d=json.load(open('gpurun_out/r3r_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])
ow=d['other_workloads']; print({r:round(v['ms'],4) for r,v in ow['mixtral_decode'].items()}, ow['qwen3_30b_a3b_prefill']['0.5']['ms'], ow['tiny']['us_per_forward'])
"
python -c "import json; d=json.load(open('gpurun_out/r3r_launches_bench_summary.json')); print(d['step_us'], [(k['kernel'][:40], k['us'], k['share']) for k in d['kernels']])"
