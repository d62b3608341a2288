mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py --scale 24 --runs 4 | tail -1; }
{
run SLPA_X=0
run SLPA_GIANT_ASYNC=0
run SLPA_X=0
} > gpurun_out/ab.log 2>&1
SLPA_TRACE=1 timeout 300 python tools/prof_run.py --scale 24 --runs 3 > gpurun_out/trace_rt.log 2>&1
