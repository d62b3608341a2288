#!/bin/bash
# A/B of builds (SLPA_LIB) and execution switches (timing only), after the parity
# tests of the default build.  Arms: "LIB:ENV=V ...".  BENCH_ARGS selects the workload.
mkdir -p gpurun_out/ab
O=gpurun_out/ab
[ -z "$SKIP_TESTS" ] && { timeout 1200 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -x -q > $O/pytest_paths.log 2>&1; echo "rc=$?" >> $O/pytest_paths.log; }
for rep in 1 2; do
for arm in "$@"; do
  lib=${arm%%:*}; envs=${arm#*:}
  echo "arm=$arm rep=$rep args=$BENCH_ARGS"
  env SLPA_LIB=$lib $envs timeout 600 python bench.py ${BENCH_ARGS:---steps 10} --warmup 3 --no-e2e --no-cpu-baseline --py-seconds 0 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],2), 'ms', {k: (v['launches'], round(v['ms'],2)) for k, v in r['profile'].items() if v['launches']})"
done
done >> $O/ab.log 2>&1
