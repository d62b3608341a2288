# Round-2 final bench lines + traffic after the last defaults changed
mkdir -p gpurun_out/final2
O=gpurun_out/final2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --mode async --py-seconds 0 > $O/bench_async.log 2>&1
timeout 600 python bench.py --variant bm --py-seconds 0 --no-cpu-baseline > $O/bench_bm.log 2>&1
timeout 600 python bench.py --graph grid --py-seconds 0 > $O/bench_grid_mg.log 2>&1
timeout 600 python bench.py --graph grid --variant bm --py-seconds 0 --no-cpu-baseline > $O/bench_grid_bm.log 2>&1
timeout 900 python bench.py --graph kmer --py-seconds 0 --no-cpu-baseline --steps 3 > $O/bench_kmer.log 2>&1
timeout 900 python bench.py --variant exact --py-seconds 0 --no-cpu-baseline --steps 3 > $O/bench_exact.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/prof_run.py --scale 24 --runs 2 --range > $O/launches.log 2>&1
timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum --cache-control none --clock-control none --csv --log-file $O/traffic.csv python tools/prof_run.py --scale 24 --runs 2 --range > $O/traffic.log 2>&1
timeout 900 python bench.py > $O/bench2.log 2>&1
