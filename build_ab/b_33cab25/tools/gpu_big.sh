# exact variant parity + scale probes (short timeouts)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or ext or xhub or move" > gpurun_out/pytest_exact.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_exact.log
timeout 300 python -c "
import time, numpy as np, paper_2411_19901_b200 as s
from oracle.oracle import get_oracle
e=s.Engine(0); e.gen_rmat(18, seed=3, permute=True)
off,tgt,w=e.download()
from tests.golden_io import GoldenGraph
g=GoldenGraph(off,tgt,w)
cfg=s.LpaConfig(variant='exact')
t=time.time(); lab,it,d,c=e.run(cfg); print('gpu exact s18', time.time()-t, it, d)
r=get_oracle().lpa_run(g,cfg); print('oracle', r.iterations, r.delta_history, np.array_equal(lab, r.labels))
for sc in (20,22,24):
    e.gen_rmat(sc, seed=2411, permute=True)
    t=time.time(); lab,it,d,c=e.run(cfg, fetch_labels=False); print('gpu exact s%d'%sc, time.time()-t, it, d, e.stats()['device_ms'], flush=True)
" > gpurun_out/exact_probe.log 2>&1
for sc in 25 26; do timeout 300 python -c "
import time, paper_2411_19901_b200 as s
t=time.time(); e=s.Engine(0); e.gen_rmat($sc, seed=2411, permute=True); print('gen s$sc', time.time()-t, e.n, e.m, flush=True)
t=time.time(); r=e.run(s.LpaConfig(), fetch_labels=False); print('run', time.time()-t, r[1], r[2], e.stats()['device_ms'], e.stats()['device_bytes']/1e9, flush=True)
" >> gpurun_out/scale_probe.log 2>&1; done
