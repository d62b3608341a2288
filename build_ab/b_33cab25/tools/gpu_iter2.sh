mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
SLPA_TRACE=1 timeout 600 python tools/e2e_probe.py 24 2>&1 | grep -v "sweep round\|L2 pers" > gpurun_out/e2e_probe.log
timeout 900 python bench.py --py-seconds 0 > gpurun_out/bench.log 2>&1
