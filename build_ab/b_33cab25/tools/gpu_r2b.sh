# Round-2: bench line + per-class profile + timeline + launch list (RMAT s24, det MG).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 env SLPA_TRACE=2 python tools/prof_run.py --scale 24 --runs 2 --profile > gpurun_out/prof24.log 2>&1
timeout 300 env SLPA_TRACE=3 python tools/prof_run.py --scale 24 --runs 2 > gpurun_out/tl24.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/launches.log 2>&1
