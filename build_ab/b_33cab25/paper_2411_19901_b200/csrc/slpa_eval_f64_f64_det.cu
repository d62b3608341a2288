// slpa_eval_f64_f64_det.cu -- evaluation kernels for weights double, sketch values double, det mode.
#include "slpa_eval.cuh"

KernelSet slpa_pick_f64_f64_det(const slpa_config *cfg) { return pick_kernels<double, true, double>(cfg); }
