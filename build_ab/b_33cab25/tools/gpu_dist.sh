mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_distributed.py -x -q -m gpu > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
