// slpa_eval_f64_f64_async.cu -- evaluation kernels for weights double, sketch values double, async mode.
#include "slpa_eval.cuh"

KernelSet slpa_pick_f64_f64_async(const slpa_config *cfg) { return pick_kernels<double, false, double>(cfg); }
