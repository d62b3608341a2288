mkdir -p gpurun_out
SLPA_BENCH_SHARE_GPU=1 SLPA_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 21 --steps 2 --warmup 1 > gpurun_out/bench_mr2.log 2>&1
timeout 600 python -m pytest tests/test_distributed.py -x -q -m gpu -k bench > gpurun_out/pytest_mr.log 2>&1; echo rc=$? >> gpurun_out/pytest_mr.log
