# A/B of execution splits and staging modes at RMAT s24 (device ms per run).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for st in 0 1; do for sp in 1 1024 2048 4096; do
  echo "=== stage $st split $sp" ; SLPA_STAGE=$st SLPA_HI_SPLIT=$sp timeout 300 python tools/prof_run.py --scale 24 --runs 3 | tail -1
done; done > gpurun_out/ab_split.log 2>&1
for st in 0 1; do for sp in 1 2048; do
  echo "=== async stage $st split $sp" ; SLPA_STAGE=$st SLPA_HI_SPLIT=$sp timeout 300 python tools/prof_run.py --scale 24 --runs 3 --mode async | tail -1
done; done >> gpurun_out/ab_split.log 2>&1
SLPA_HI_SPLIT=2048 timeout 300 python tools/prof_run.py --scale 24 --runs 2 --profile > gpurun_out/prof_2048.log 2>&1
