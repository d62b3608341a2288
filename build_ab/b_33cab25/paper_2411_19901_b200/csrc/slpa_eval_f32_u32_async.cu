// slpa_eval_f32_u32_async.cu -- evaluation kernels for weights float, sketch values uint32_t, async mode.
#include "slpa_eval.cuh"

KernelSet slpa_pick_f32_u32_async(const slpa_config *cfg) { return pick_kernels<float, false, uint32_t>(cfg); }
