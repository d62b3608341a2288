// slpa_eval_f32_f64_det.cu -- evaluation kernels for weights float, sketch values double, det mode.
#include "slpa_eval.cuh"

KernelSet slpa_pick_f32_f64_det(const slpa_config *cfg) { return pick_kernels<float, true, double>(cfg); }
