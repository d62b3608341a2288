# Round bench + evidence: full GPU tests, smoke, default bench line, variants / configs, reference arm,
# ncu launch list, ncu traffic per class, full capture of the top kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/clocks_pre.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --mode async --no-cpu-baseline > gpurun_out/bench_async.log 2>&1
timeout 600 python bench.py --variant bm --no-cpu-baseline > gpurun_out/bench_bm.log 2>&1
timeout 600 python bench.py --graph grid --no-cpu-baseline > gpurun_out/bench_grid_mg.log 2>&1
timeout 600 python bench.py --graph grid --variant bm --no-cpu-baseline > gpurun_out/bench_grid_bm.log 2>&1
timeout 900 python bench.py --graph kmer --no-cpu-baseline --steps 3 > gpurun_out/bench_kmer.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/launches.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic.csv -k regex:"k_mg_hi_scan|k_mg_hi_merge|k_mg_hi_finish|k_mg_hi_block|k_lane_direct|k_lo_warp|k_mg_giant_grp|k_giant_gather" python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/traffic.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mg_hi_scan" -c 1 -o gpurun_out/full_top python tools/prof_run.py --scale 24 --runs 1 > gpurun_out/full_top.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_lane_direct" -c 1 -o gpurun_out/full_kmer python tools/prof_run.py --graph kmer --scale 27 --runs 1 > /dev/null 2>&1
