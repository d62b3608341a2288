// slpa_eval_f32_f64_async.cu -- evaluation kernels for weights float, sketch values double, async mode.
#include "slpa_eval.cuh"

KernelSet slpa_pick_f32_f64_async(const slpa_config *cfg) { return pick_kernels<float, false, double>(cfg); }
