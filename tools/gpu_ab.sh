mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -k async 2>&1 | tail -2
timeout 600 python -m pytest tests/test_distributed.py -x -q -m gpu 2>&1 | tail -2
} > gpurun_out/ab.log 2>&1
