# A/B of heavy-scan variants (eval ms per run, RMAT s24 det) + ncu of the pipe kernel.
mkdir -p gpurun_out
run() { echo "=== $*"; env "$@" timeout 300 python tools/prof_run.py --scale 24 --runs 2 --profile 2>&1 | grep -E "^run 1|eval_hi_rk|eval_giant|eval_lo"; }
{
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
run SLPA_HI_SCAN=2
run SLPA_HI_SCAN=0
} > gpurun_out/ab.log 2>&1
bash tools/gpu_ncu1.sh k_mg_hi_pipe
