# ncu full capture of one kernel (first launch) on RMAT s24: $1 = kernel regex, rest = env
mkdir -p gpurun_out
K=$1; shift
env "$@" timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"$K" -c 1 -o gpurun_out/full_$K -f python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/full_$K.log 2>&1
