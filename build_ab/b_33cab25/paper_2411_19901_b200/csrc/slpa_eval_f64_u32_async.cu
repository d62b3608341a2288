// slpa_eval_f64_u32_async.cu -- evaluation kernels for weights double, sketch values uint32_t, async mode.
#include "slpa_eval.cuh"

KernelSet slpa_pick_f64_u32_async(const slpa_config *cfg) { return pick_kernels<double, false, uint32_t>(cfg); }
