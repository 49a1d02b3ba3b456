python -c "from paper_2507_17133_b200.build import build; build()"
timeout 1500 python scripts/ab.py --env BO_H_PAD=64 --env BO_H_PAD=256 --env BO_H_PAD=512 --workloads mixtral_decode:1.0,mixtral_decode:0.0,mixtral_prefill:0.5,qwen3_30b_a3b_prefill:0.5 --reps 6 > gpurun_out/r2z_ab_hpad.json 2> gpurun_out/r2z_ab_hpad.err
cat gpurun_out/r2z_pytest_hpad.log
python - <<'P'
import json
d=json.load(open("gpurun_out/r2z_ab_hpad.json"))
for wl,v in d.items():
    if wl=="arms": continue
    for arm,r in v.items():
        print(wl,arm,r["ms_median"],r["kernel_ms"])
P
