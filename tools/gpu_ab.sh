# A/B: heavy chunk streaming flavours (device ms per run + first k_mg_hi_scan launch, RMAT s24 det)
mkdir -p gpurun_out
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py --scale 24 --runs 5 2>&1 | grep -E "^run [234]"; env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__inst_executed.sum --clock-control none --cache-control none -k regex:k_mg_hi_scan -c 1 python tools/prof_run.py --scale 24 --runs 1 2>&1 | grep -E "gpu__time|dram__bytes|inst_exec"; }
{
run SLPA_STREAM=1
run SLPA_STREAM=2
run SLPA_STREAM=0
} > gpurun_out/ab.log 2>&1
