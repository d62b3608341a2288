mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py tests/test_distributed.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py --scale 24 --runs 4 | tail -1; }
{
run SLPA_X=0
run SLPA_LO_SMALL=0
run SLPA_HI_SMALL=0
run SLPA_LO_SMALL=8192 SLPA_HI_SMALL=32768
run SLPA_X=0
} > gpurun_out/ab.log 2>&1
SLPA_TRACE=3 timeout 300 python tools/prof_run.py --scale 24 --runs 2 > gpurun_out/tl.log 2>&1
