O=gpurun_out/r2g; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
SKIP_TESTS=1 bash tools/gpu_ab.sh ":" "build_ab/lo1.so:"
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --mode async --py-seconds 0 > $O/bench_async.log 2>&1
timeout 600 python bench.py --variant bm --py-seconds 0 --no-cpu-baseline > $O/bench_bm.log 2>&1
timeout 600 python bench.py --graph grid --py-seconds 0 > $O/bench_grid_mg.log 2>&1
timeout 600 python bench.py --graph grid --variant bm --py-seconds 0 --no-cpu-baseline > $O/bench_grid_bm.log 2>&1
timeout 900 python bench.py --graph kmer --py-seconds 0 --no-cpu-baseline --steps 3 > $O/bench_kmer.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations 15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
