// slpa_eval_f64_u32_det.cu -- evaluation kernels for weights double, sketch values uint32_t, det mode.
#include "slpa_eval.cuh"

KernelSet slpa_pick_f64_u32_det(const slpa_config *cfg) { return pick_kernels<double, true, uint32_t>(cfg); }
