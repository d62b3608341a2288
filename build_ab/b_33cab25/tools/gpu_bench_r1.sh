set -x
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/clocks_pre.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r1.log 2>&1
timeout 600 python bench.py --mode async --no-cpu-baseline > gpurun_out/bench_r1_async.log 2>&1
timeout 600 python bench.py --variant bm --no-cpu-baseline > gpurun_out/bench_r1_bm.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_r1.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_mg_hi_win|k_lane_win" -s 0 -c 2 -o gpurun_out/full_r1 python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/full_r1.log 2>&1
