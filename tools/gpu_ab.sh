mkdir -p gpurun_out
{
echo "=== now det"; timeout 300 python tools/prof_run.py --scale 24 --runs 6 2>&1 | grep -E "^run [2345]"
echo "=== now async"; timeout 300 python tools/prof_run.py --scale 24 --runs 4 --mode async 2>&1 | grep -E "^run [23]"
echo "=== now kmer"; timeout 300 python tools/prof_run.py --graph kmer --scale 27 --runs 3 2>&1 | grep -E "^run [2]"
echo "=== now kmer lo0"; SLPA_LO_DIRECT=0 timeout 300 python tools/prof_run.py --graph kmer --scale 27 --runs 3 2>&1 | grep -E "^run [2]"
echo "=== now grid"; timeout 300 python tools/prof_run.py --graph grid --scale 24 --runs 4 2>&1 | grep -E "^run [23]"
echo "=== old grid"; (cd build_ab/old && timeout 300 python tools/prof_run.py --graph grid --scale 24 --runs 4 2>&1 | grep -E "^run [23]")
} > gpurun_out/ab.log 2>&1
