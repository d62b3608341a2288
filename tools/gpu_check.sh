#!/bin/bash
# HEAD check on one B200: GPU suite, smoke, default bench line.
mkdir -p gpurun_out/chk
O=gpurun_out/chk
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --py-seconds 0 > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
timeout 2400 python -m pytest tests -m gpu -x -q --durations 15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
