mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py --scale 24 --runs 3 | tail -1; }
{
run SLPA_X=0
run SLPA_STREAM=0
run SLPA_GIANT=65536
run SLPA_GIANT=32768
run SLPA_L2_PERSIST_MB=30
run SLPA_L2_PERSIST_MB=60
run SLPA_L2_PERSIST_MB=100
run SLPA_L2_PERSIST_MB=60 SLPA_GIANT=65536
echo "=== async"; timeout 300 python tools/prof_run.py --scale 24 --runs 3 --mode async | tail -1
echo "=== async L2 60"; SLPA_L2_PERSIST_MB=60 timeout 300 python tools/prof_run.py --scale 24 --runs 3 --mode async | tail -1
} > gpurun_out/ab.log 2>&1
SLPA_TRACE=1 SLPA_L2_PERSIST_MB=60 timeout 300 python tools/prof_run.py --scale 24 --runs 1 2>&1 | grep "L2" > gpurun_out/l2.log
