python -c "from paper_2507_17133_b200.build import build; build(); build(variant='probe')"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_router_exact.py tests/test_gpu_shared.py tests/test_gpu_swap_tail.py tests/test_gpu_distill.py -m gpu -q -x --timeout 600 2>&1 | tail -5 > gpurun_out/r2n_pytest.log
BO_LIB=probe timeout 300 python scripts/probe_tiles.py qwen3_30b_a3b_prefill 0.5 > gpurun_out/r2n_probe_c4.json 2> gpurun_out/r2n_probe.err
BO_LIB=probe timeout 300 python scripts/probe_tiles.py mixtral_prefill 0.5 > gpurun_out/r2n_probe_c2.json 2>> gpurun_out/r2n_probe.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
tail -3 gpurun_out/r2n_pytest.log
