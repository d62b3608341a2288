# First k_mg_hi_scan launch: pipeline depth variants (timing experiment)
mkdir -p gpurun_out
one() { tag=$1; shift; env "$@" timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__warps_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control none -k regex:k_mg_hi_scan -c 1 python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/ab_$tag.log 2>&1; }
one s1 SLPA_STREAM=1
one s2 SLPA_STREAM=2
one s1b SLPA_STREAM=1 SLPA_LIB=build_ab/lib_minb2.so
one s2b SLPA_STREAM=2 SLPA_LIB=build_ab/lib_minb2.so
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py --scale 24 --runs 3 2>&1 | grep -E "^run 2"; }
{
run SLPA_STREAM=1
run SLPA_STREAM=2
run SLPA_STREAM=1 SLPA_LIB=build_ab/lib_minb2.so
run SLPA_STREAM=2 SLPA_LIB=build_ab/lib_minb2.so
} > gpurun_out/ab.log 2>&1
