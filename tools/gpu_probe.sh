mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
SLPA_TRACE=1 timeout 600 python tools/e2e_prof.py --scale 24 --reps 4 2>&1 | grep -v "sweep round\|L2 pers" > gpurun_out/e2e.log 2>&1
