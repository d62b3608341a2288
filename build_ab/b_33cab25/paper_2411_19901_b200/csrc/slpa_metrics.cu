// slpa_metrics.cu -- community tallies and modularity on the device
// (metrics.py:34-74).  One pass over the arcs: each vertex reduces its own
// row (incident weight, weight to same-label neighbours) and issues three
// atomics into label-indexed float64 / int64 tallies; a second pass reduces
// Q = sum_c internal_c/total - (incident_c/total)^2.  float64 throughout,
// like the reference; summation order differs from np.bincount, so results
// agree to ~1e-15 relative (tests use 1e-9, as test_metrics.py:43-50 does).
#include <algorithm>
#include "slpa_internal.cuh"

namespace {
constexpr int kT = 256;
constexpr int64_t kWarpDeg = 128;  // rows at least this long are reduced by a warp

__global__ void k_check_labels(const int32_t *lab, int64_t n, unsigned *err) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && (lab[i] < 0 || lab[i] >= n)) atomicOr(err, 1u);
}

template <class W>
__global__ void __launch_bounds__(kT) k_tally_rows(const int64_t *__restrict__ off, const int32_t *__restrict__ tgt,
                                                   const W *__restrict__ w, const int32_t *__restrict__ lab, int64_t n,
                                                   double *internal, double *incident, unsigned long long *sizes,
                                                   int64_t v0, int64_t v1) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int32_t L = lab[v];
    if (v >= v0 && v < v1) atomicAdd(&sizes[L], 1ull);  // owned vertices (partitioned tallies)
    const int64_t lo = off[v], hi = off[v + 1];
    if (hi - lo >= kWarpDeg || hi == lo) return;
    double inc = 0.0, in = 0.0;
    for (int64_t e = lo; e < hi; ++e) {
        double x = (double)__ldg(&w[e]);
        inc += x;
        if (__ldg(&lab[__ldg(&tgt[e])]) == L) in += x;
    }
    atomicAdd(&incident[L], inc);
    if (in != 0.0) atomicAdd(&internal[L], in);
}

template <class W>
__global__ void __launch_bounds__(kT) k_tally_rows_warp(const int64_t *__restrict__ off,
                                                        const int32_t *__restrict__ tgt, const W *__restrict__ w,
                                                        const int32_t *__restrict__ lab, int64_t n, double *internal,
                                                        double *incident) {
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
        const int64_t lo = off[v], hi = off[v + 1];
        if (hi - lo < kWarpDeg) continue;
        const int32_t L = lab[v];
        double inc = 0.0, in = 0.0;
        for (int64_t e = lo + lane; e < hi; e += 32) {
            double x = (double)__ldg(&w[e]);
            inc += x;
            if (__ldg(&lab[__ldg(&tgt[e])]) == L) in += x;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            inc += __shfl_xor_sync(0xffffffffu, inc, o);
            in += __shfl_xor_sync(0xffffffffu, in, o);
        }
        if (lane == 0) {
            atomicAdd(&incident[L], inc);
            if (in != 0.0) atomicAdd(&internal[L], in);
        }
    }
}

// pass 1: total = sum incident, ncomm = #sizes > 0; pass 2: Q terms
__global__ void __launch_bounds__(kT) k_reduce_total(const double *incident, const unsigned long long *sizes,
                                                     int64_t n, double *total, unsigned long long *ncomm) {
    __shared__ double sd[kT / 32];
    __shared__ unsigned long long sc[kT / 32];
    double acc = 0.0;
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        acc += incident[i];
        c += sizes[i] > 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0) { sd[threadIdx.x >> 5] = acc; sc[threadIdx.x >> 5] = c; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        unsigned long long u = 0;
        for (int i = 0; i < kT / 32; ++i) { t += sd[i]; u += sc[i]; }
        atomicAdd(total, t);
        atomicAdd(ncomm, u);
    }
}
__global__ void __launch_bounds__(kT) k_reduce_q(const double *internal, const double *incident, int64_t n,
                                                 const double *total, double *q) {
    __shared__ double sd[kT / 32];
    const double tot = *total;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double f = incident[i] / tot;
        acc += internal[i] / tot - f * f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sd[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < kT / 32; ++i) t += sd[i];
        atomicAdd(q, t);
    }
}
}  // namespace

// d_lab: labels by position (active numbering); label values are vertex ids.
void slpa_tally(slpa_ctx *ctx, const int32_t *d_lab, double *q, int64_t *ncomm, int64_t *sizes, double *internal,
                double *incident) {
    DeviceGraph &g = ctx->g;
    WorkBuffers &wb = ctx->wb;
    cudaStream_t s = ctx->stream;
    const int64_t n = g.n;
    wb.metric_d.alloc(2 * n + 2);
    wb.metric_u.alloc(n + 2);
    double *d_int = wb.metric_d.p, *d_inc = wb.metric_d.p + n, *d_tot = wb.metric_d.p + 2 * n,
           *d_q = wb.metric_d.p + 2 * n + 1;
    const int64_t v0 = ctx->part ? ctx->v_begin : 0, v1 = ctx->part ? ctx->v_end : n;
    unsigned long long *d_sz = wb.metric_u.p, *d_nc = wb.metric_u.p + n;
    unsigned *d_err = (unsigned *)(wb.metric_u.p + n + 1);
    CUDA_TRY(cudaMemsetAsync(wb.metric_d.p, 0, (2 * n + 2) * sizeof(double), s));
    CUDA_TRY(cudaMemsetAsync(wb.metric_u.p, 0, (n + 2) * sizeof(unsigned long long), s));
    if (n > 0) k_check_labels<<<grid_for(n, kT), kT, 0, s>>>(d_lab, n, d_err);
    unsigned err = 0;
    CUDA_TRY(cudaMemcpyAsync(&err, d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (err) throw SlpaError{SLPA_EINVAL, "label out of range"};
    if (n > 0) {
        const unsigned wgrid = (unsigned)std::min<int64_t>((n * 32 + kT - 1) / kT, 148 * 32);
        if (g.w_f64) {
            k_tally_rows<double><<<grid_for(n, kT), kT, 0, s>>>(g.off(), g.tgt(), (const double *)g.w(), d_lab, n,
                                                                d_int, d_inc, d_sz, v0, v1);
            k_tally_rows_warp<double><<<wgrid, kT, 0, s>>>(g.off(), g.tgt(), (const double *)g.w(), d_lab, n, d_int,
                                                           d_inc);
        } else {
            k_tally_rows<float><<<grid_for(n, kT), kT, 0, s>>>(g.off(), g.tgt(), (const float *)g.w(), d_lab, n, d_int,
                                                               d_inc, d_sz, v0, v1);
            k_tally_rows_warp<float><<<wgrid, kT, 0, s>>>(g.off(), g.tgt(), (const float *)g.w(), d_lab, n, d_int,
                                                          d_inc);
        }
        const unsigned rgrid = (unsigned)std::min<int64_t>(grid_for(n, kT), 148 * 8);
        k_reduce_total<<<rgrid, kT, 0, s>>>(d_inc, d_sz, n, d_tot, d_nc);
        CUDA_TRY(cudaGetLastError());
    }
    double tot = 0.0;
    unsigned long long nc = 0;
    CUDA_TRY(cudaMemcpyAsync(&tot, d_tot, sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&nc, d_nc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (ncomm) *ncomm = (int64_t)nc;
    if (sizes) CUDA_TRY(cudaMemcpyAsync(sizes, d_sz, n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    if (internal) CUDA_TRY(cudaMemcpyAsync(internal, d_int, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (incident) CUDA_TRY(cudaMemcpyAsync(incident, d_inc, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (q) {
        if (!(tot > 0.0)) {
            CUDA_TRY(cudaStreamSynchronize(s));
            throw SlpaError{SLPA_EINVAL, "modularity is undefined on a graph with no edges"};
        }
        const unsigned rgrid = (unsigned)std::min<int64_t>(grid_for(n, kT), 148 * 8);
        k_reduce_q<<<rgrid, kT, 0, s>>>(d_int, d_inc, n, d_tot, d_q);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(q, d_q, sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------ partitioned
namespace {
__global__ void __launch_bounds__(kT) k_sum(const double *x, int64_t n, double *out) {
    __shared__ double sd[kT / 32];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += x[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sd[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < kT / 32; ++i) t += sd[i];
        atomicAdd(out, t);
    }
}
__global__ void __launch_bounds__(kT) k_sum_sq_frac(const double *x, int64_t n, const double *tot, double *out) {
    __shared__ double sd[kT / 32];
    const double t = *tot;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double f = x[i] / t;
        acc += f * f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sd[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int i = 0; i < kT / 32; ++i) a += sd[i];
        atomicAdd(out, a);
    }
}
}  // namespace

// Rank-local tallies over the owned rows with the full label replica:
// incident / sizes stay on the device (metric buffers) for an all-reduce;
// the internal weight is returned as a scalar (sum over communities is
// additive, so only its total is needed for Q).
void slpa_part_tally_impl(slpa_ctx *ctx, double *internal_local, uint64_t *incident_dptr, uint64_t *sizes_dptr) {
    const int64_t n = ctx->g.n;
    slpa_tally(ctx, ctx->wb.lab_old.p, nullptr, nullptr, nullptr, nullptr, nullptr);
    DevBuf<double> acc;
    acc.alloc(1);
    CUDA_TRY(cudaMemsetAsync(acc.p, 0, sizeof(double), ctx->stream));
    const unsigned rgrid = (unsigned)std::min<int64_t>(grid_for(std::max<int64_t>(n, 1), kT), 148 * 8);
    if (n > 0) k_sum<<<rgrid, kT, 0, ctx->stream>>>(ctx->wb.metric_d.p, n, acc.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(internal_local, acc.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    acc.release();
    *incident_dptr = (uint64_t)(uintptr_t)(ctx->wb.metric_d.p + n);
    *sizes_dptr = (uint64_t)(uintptr_t)ctx->wb.metric_u.p;
}

// Q = internal_total / total - sum_c (incident_c / total)^2 on the summed
// incident array (metrics.py:70-74).
void slpa_part_modularity_impl(slpa_ctx *ctx, double internal_total, double *q) {
    const int64_t n = ctx->g.n;
    const double *inc = ctx->wb.metric_d.p + n;
    DevBuf<double> acc;
    acc.alloc(2);
    CUDA_TRY(cudaMemsetAsync(acc.p, 0, 2 * sizeof(double), ctx->stream));
    const unsigned rgrid = (unsigned)std::min<int64_t>(grid_for(std::max<int64_t>(n, 1), kT), 148 * 8);
    if (n > 0) k_sum<<<rgrid, kT, 0, ctx->stream>>>(inc, n, acc.p);
    double tot = 0.0;
    CUDA_TRY(cudaMemcpyAsync(&tot, acc.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (!(tot > 0.0)) {
        acc.release();
        throw SlpaError{SLPA_EINVAL, "modularity is undefined on a graph with no edges"};
    }
    if (n > 0) k_sum_sq_frac<<<rgrid, kT, 0, ctx->stream>>>(inc, n, acc.p, acc.p + 1);
    double sq = 0.0;
    CUDA_TRY(cudaMemcpyAsync(&sq, acc.p + 1, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    acc.release();
    *q = internal_total / tot - sq;
}
