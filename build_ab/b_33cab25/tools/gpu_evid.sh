# Evidence: ncu traffic per family (one lpa_run, no cache flush), sanitizers, exact timing, s27 generation probe.
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum --cache-control none --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/prof_run.py --scale 24 --runs 2 --range > gpurun_out/traffic.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_run.py --scale 24 --runs 2 --range > gpurun_out/launches.log 2>&1
for mode in det async; do
timeout 600 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/prof_run.py --scale 12 --runs 1 --mode $mode > gpurun_out/memcheck_$mode.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_$mode.log
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/prof_run.py --scale 12 --runs 1 --mode $mode > gpurun_out/racecheck_$mode.log 2>&1; echo "rc=$?" >> gpurun_out/racecheck_$mode.log
done
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/prof_run.py --scale 12 --runs 1 --variant bm > gpurun_out/memcheck_bm.log 2>&1; echo "rc=$?" >> gpurun_out/memcheck_bm.log
timeout 300 python -c "
import sys, time, numpy as np
sys.path.insert(0, 'tests')
import paper_2411_19901_b200 as s
from oracle.oracle import get_oracle
from golden_io import GoldenGraph
e=s.Engine(0); e.gen_rmat(18, seed=3, permute=True)
off,tgt,w=e.download(); g=GoldenGraph(off,tgt,w)
cfg=s.LpaConfig(variant='exact')
t=time.time(); lab,it,d,c=e.run(cfg); print('gpu exact s18', time.time()-t, it, d)
r=get_oracle().lpa_run(g,cfg); print('oracle', r.iterations, r.delta_history, np.array_equal(lab, r.labels))
for sc in (20,22,24):
    e.gen_rmat(sc, seed=2411, permute=True)
    t=time.time(); lab,it,d,c=e.run(cfg, fetch_labels=False); print('gpu exact s%d'%sc, time.time()-t, it, d, e.stats()['device_ms'], flush=True)
" > gpurun_out/exact_probe.log 2>&1
timeout 400 python -c "
import time, paper_2411_19901_b200 as s
t=time.time(); e=s.Engine(0); e.gen_rmat(27, seed=2411, permute=True); print('gen s27', time.time()-t, e.n, e.m, flush=True)
t=time.time(); r=e.run(s.LpaConfig(), fetch_labels=False); print('run', time.time()-t, r[1], r[2], e.stats()['device_ms'], e.stats()['device_bytes']/1e9, flush=True)
" > gpurun_out/s27_probe.log 2>&1; echo "rc=$?" >> gpurun_out/s27_probe.log
