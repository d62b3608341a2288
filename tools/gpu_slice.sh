#!/bin/bash
# Heavy-slice A/B (repeated) + timeline at s24 + the distributed GPU tests.
mkdir -p gpurun_out
{
for rep in 1 2; do
  for sl in 65536 131072 262144 524288; do
    echo "rep=$rep slice=$sl"
    SLPA_HI_SLICE=$sl timeout 600 python bench.py --scale 24 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --py-seconds 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],2), 'ms', {k: round(v['ms'],1) for k, v in r['families'].items()}, 'B/vertex', round(d['memory']['engine_bytes_per_vertex'],1))"
  done
done
} > gpurun_out/slice.log 2>&1
SLPA_TRACE=3 timeout 300 python -u tools/prof_run.py --scale 24 --runs 2 > gpurun_out/tl24.log 2>&1
timeout 900 python -m pytest tests/test_distributed.py -x -q -m gpu > gpurun_out/dist.log 2>&1
