mkdir -p gpurun_out
{
echo "=== now det"; timeout 300 python tools/prof_run.py --scale 24 --runs 5 2>&1 | grep -E "^run [234]"
echo "=== now async"; timeout 300 python tools/prof_run.py --scale 24 --runs 4 --mode async 2>&1 | grep -E "^run [23]"
echo "=== old async"; (cd build_ab/old && timeout 300 python tools/prof_run.py --scale 24 --runs 4 --mode async 2>&1 | grep -E "^run [23]")
echo "=== now kmer"; timeout 300 python tools/prof_run.py --graph kmer --scale 27 --runs 3 2>&1 | grep -E "^run [2]"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
} > gpurun_out/ab.log 2>&1
