# Full GPU suite + smoke + default bench + reference arm + variants (round-2 evidence)
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/clocks_pre.txt
timeout 2400 python -m pytest tests -m gpu -x -q --durations 15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 600 python bench.py --mode async --py-seconds 0 > gpurun_out/bench_async.log 2>&1
timeout 600 python bench.py --variant bm --py-seconds 0 --no-cpu-baseline > gpurun_out/bench_bm.log 2>&1
timeout 600 python bench.py --graph grid --py-seconds 0 > gpurun_out/bench_grid_mg.log 2>&1
timeout 600 python bench.py --graph grid --variant bm --py-seconds 0 --no-cpu-baseline > gpurun_out/bench_grid_bm.log 2>&1
timeout 900 python bench.py --graph kmer --py-seconds 0 --no-cpu-baseline --steps 3 > gpurun_out/bench_kmer.log 2>&1
timeout 900 python bench.py --variant exact --py-seconds 0 --no-cpu-baseline --steps 3 > gpurun_out/bench_exact.log 2>&1
