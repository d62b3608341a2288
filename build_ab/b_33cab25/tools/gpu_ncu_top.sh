# ncu: launch list of one lpa_run + full capture of the first k_mg_hi_scan launch (RMAT s24)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"${1:-k_mg_hi_scan}" -c 1 -o gpurun_out/full_top -f python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/full_top.log 2>&1
