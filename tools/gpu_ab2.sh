#!/bin/bash
# A/B of alternative builds (SLPA_LIB) on the bench workloads; timing only.
mkdir -p gpurun_out
for lib in "" build_ab/ef.so build_ab/minb3.so; do
  for sc in 24 27; do
    st=10; [ $sc = 27 ] && st=3
    echo "lib=${lib:-default} scale=$sc"
    SLPA_LIB=$lib timeout 600 python bench.py --scale $sc --steps $st --warmup 3 --no-e2e --no-cpu-baseline --py-seconds 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],2), 'ms', {k: round(v['ms'],1) for k, v in r['families'].items()})"
  done
done > gpurun_out/ab2.log 2>&1
