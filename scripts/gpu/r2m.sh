python -c "from paper_2507_17133_b200.build import build; build(); build(variant='probe')"
REPS=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_route_fused" --launch-skip 1 --launch-count 1 -o gpurun_out/r2m_route_fused python scripts/ffn_ncu_ab.py mixtral_decode 1.0 > gpurun_out/r2m_ncu_rf.log 2>&1
BO_LIB=probe timeout 300 python scripts/probe_tiles.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r2m_probe_c4.json 2> gpurun_out/r2m_probe.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_prefill 0.5 > gpurun_out/r2m_probe_c2.json 2>> gpurun_out/r2m_probe.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_decode 1.0 > gpurun_out/r2m_probe_c3r1.json 2>> gpurun_out/r2m_probe.err
tail -3 gpurun_out/r2m_ncu_rf.log
