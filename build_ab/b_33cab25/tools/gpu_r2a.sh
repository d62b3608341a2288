# Round-2 first check: GPU tests, smoke, default bench line, reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/clocks_pre.txt
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations 20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
