# EP on the GPU: device tables, virtual EP, graph capture, 2-process gloo, NCCL world 1; C client; api
python -c "from paper_2507_17133_b200.build import build; build()"
timeout 1500 python -m pytest tests/test_ep.py tests/test_c_client.py tests/test_gpu_api.py -m gpu -q -x 2>&1 | tail -40 > gpurun_out/r2c_pytest_ep.log
BO_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 4 --warmup 3 --workload mixtral_decode --no-sweep > gpurun_out/r2c_bench_ep2_gloo.json 2> gpurun_out/r2c_bench_ep2_gloo.err
tail -3 gpurun_out/r2c_pytest_ep.log
