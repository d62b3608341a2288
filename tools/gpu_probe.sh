mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py $G --runs 5 | tail -1; }
{
G="--scale 24"; run SLPA_X=0; run SLPA_X=0
G="--scale 24 --mode async"; run SLPA_X=0
} > gpurun_out/ab.log 2>&1
