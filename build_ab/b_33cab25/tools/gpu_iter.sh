# Iteration check: fast parity tests, bench line, timeline.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
timeout 900 python bench.py --py-seconds 0 > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --graph kmer --py-seconds 0 --no-cpu-baseline --steps 3 > gpurun_out/bench_kmer.log 2>&1
timeout 300 env SLPA_TRACE=3 python tools/prof_run.py --scale 24 --runs 2 > gpurun_out/tl24.log 2>&1
