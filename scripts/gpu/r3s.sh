# decode GEMM2 split-K at every ratio (few tiles on 148 SMs at ratio 0.5): interleaved A/B + launch lists
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 900 python scripts/ab.py --env BO_GEMM2_SPLITK=1 --workloads mixtral_decode:0.5,mixtral_decode:0.25,mixtral_decode:0.0,mixtral_decode:0.75 --reps 8 > gpurun_out/r3s_ab_splitk.json 2> gpurun_out/r3s_ab_splitk.err
for arm in 0 1; do
  REPS=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/ffn_ncu_ab.py mixtral_decode 0.5 BO_GEMM2_SPLITK=$arm > gpurun_out/r3s_launches_c3r05_s$arm.csv 2> gpurun_out/r3s_launches_c3r05_s$arm.err
  python scripts/launch_summary.py gpurun_out/r3s_launches_c3r05_s$arm.csv > gpurun_out/r3s_launches_c3r05_s${arm}_summary.json
done
python - <<'P'
import json
d=json.load(open("gpurun_out/r3s_ab_splitk.json"))
for wl,v in d.items():
    if wl=="arms": continue
    for arm,r in v.items():
        print(wl,arm,r["ms_median"],{k:round(x*1000,1) for k,x in r["kernel_ms"].items()})
P
for f in gpurun_out/r3s_launches_*_summary.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['step_us'], [(k['kernel'][:40], k['us']) for k in d['kernels']])"; done
