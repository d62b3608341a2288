mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_distributed.py -m gpu -x -q > gpurun_out/pytest_dist.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dist.log
