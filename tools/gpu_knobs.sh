#!/bin/bash
# Env-knob sweep (timing only) at RMAT s27 and s24.
mkdir -p gpurun_out
for sc in 27 24; do
  st=10; [ $sc = 27 ] && st=3
  for env in "" "SLPA_DEFER_MIN=0" "SLPA_DEFER_MIN=20000" "SLPA_DEFER_MIN=200000" "SLPA_DEFER_MIN=2000000" \
             "SLPA_HI_SLICE=262144" "SLPA_HI_SLICE=16384" "SLPA_GIANT=65536" "SLPA_GIANT=16384" "SLPA_DEFER=1"; do
    echo "scale=$sc env=${env:-default}"
    env $env timeout 600 python bench.py --scale $sc --steps $st --warmup 3 --no-e2e --no-cpu-baseline --py-seconds 0 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; s=d['run_stats']; print(round(d['ms_per_step'],2), 'ms', {k: round(v['ms'],1) for k, v in r['families'].items()}, 'rounds', round(s['rounds'],1), 'arc_reads', '%.3g' % s['arc_reads'])"
  done
done > gpurun_out/knobs.log 2>&1
