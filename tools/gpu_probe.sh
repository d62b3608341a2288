mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py --scale 24 --runs 3 | tail -1; }
{
run SLPA_X=0
run SLPA_GIANT_GRP=0
run SLPA_GIANT=16384
run SLPA_GIANT=4096
echo "=== async"; timeout 300 python tools/prof_run.py --scale 24 --runs 3 --mode async | tail -1
} > gpurun_out/ab.log 2>&1
SLPA_TRACE=1 timeout 300 python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/trace.log 2>&1
timeout 300 python tools/prof_run.py --scale 24 --runs 2 --profile > gpurun_out/prof.log 2>&1
