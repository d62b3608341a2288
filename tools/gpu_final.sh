#!/bin/bash
# Round-end evidence on one B200: GPU suite, smoke, bench lines (all configs / modes /
# variants, reference arm, N=2 protocol run), ncu launch list / DRAM traffic / full
# captures of the two hot kernels.
O=${1:-gpurun_out/final}
mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $O/clocks_pre.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1
timeout 600 python bench.py --mode async --py-seconds 0 > $O/bench_async.log 2>&1
timeout 600 python bench.py --variant bm --py-seconds 0 --no-cpu-baseline > $O/bench_bm.log 2>&1
timeout 600 python bench.py --graph grid --py-seconds 0 > $O/bench_grid_mg.log 2>&1
timeout 600 python bench.py --graph grid --variant bm --py-seconds 0 --no-cpu-baseline > $O/bench_grid_bm.log 2>&1
timeout 900 python bench.py --graph kmer --py-seconds 0 --no-cpu-baseline --steps 3 > $O/bench_kmer.log 2>&1
timeout 900 python bench.py --variant exact --py-seconds 0 --no-cpu-baseline --steps 3 > $O/bench_exact.log 2>&1
timeout 900 python bench.py --scale 27 --py-seconds 0 --no-cpu-baseline --no-e2e --steps 3 > $O/bench_s27.log 2>&1
SLPA_BENCH_SHARE_GPU=1 SLPA_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --scale 21 --steps 2 --warmup 3 > $O/bench_mr2.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/prof_run.py --scale 24 --runs 2 --range > $O/launches.log 2>&1
timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum --cache-control none --clock-control none --csv --log-file $O/traffic.csv python tools/prof_run.py --scale 24 --runs 2 --range > $O/traffic.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_mg_hi_scan -c 1 -o $O/full_hi_scan -f python tools/prof_run.py --scale 24 --runs 1 > $O/full_hi_scan.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_lane_direct -c 1 -o $O/full_lane -f python tools/prof_run.py --scale 24 --runs 1 > $O/full_lane.log 2>&1
# (compute-sanitizer is closed on the GPU pool; profiles/r2_sanitizer.md holds the earlier memcheck / racecheck runs)
timeout 2400 python -m pytest tests -m gpu -x -q --durations 15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
