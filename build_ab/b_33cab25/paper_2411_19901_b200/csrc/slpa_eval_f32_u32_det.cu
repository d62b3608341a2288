// slpa_eval_f32_u32_det.cu -- evaluation kernels for weights float, sketch values uint32_t, det mode.
#include "slpa_eval.cuh"

KernelSet slpa_pick_f32_u32_det(const slpa_config *cfg) { return pick_kernels<float, true, uint32_t>(cfg); }
