# A/B: L2 persisting set-aside for the label words (device ms per run, RMAT s24 det)
mkdir -p gpurun_out
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py --scale 24 --runs 4 2>&1 | grep -E "^run [23]"; }
{
run SLPA_L2_PERSIST_MB=4096
run SLPA_L2_PERSIST_MB=0
run SLPA_L2_PERSIST_MB=32
run SLPA_L2_PERSIST_MB=48
} > gpurun_out/ab.log 2>&1
