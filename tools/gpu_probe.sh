mkdir -p gpurun_out
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py $G --runs 6 | tail -2; }
{
G="--scale 24"; run SLPA_X=0; run SLPA_GIANT=65536; run SLPA_GIANT=131072; run SLPA_GIANT=262144; run SLPA_X=0
} > gpurun_out/ab.log 2>&1
