#!/bin/bash
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --py-seconds 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],2), 'ms', {k: (v['launches'], round(v['ms'],2)) for k, v in r['profile'].items()})"; done
} > gpurun_out/commit.log 2>&1
SLPA_TRACE=3 timeout 300 python -u tools/prof_run.py --scale 24 --runs 2 > gpurun_out/tl24b.log 2>&1
