// slpa_validate.cu -- validate_graph (graph.py:378-403) on the device.
//
// The reference checks, in this order: strictly increasing neighbour lists
// (first offending vertex named), positive weights, exact arc symmetry with
// equal reverse weights (lexsort of the reversed arc list), and the
// degree-sum identity sum_i weighted_degree(i) == 2 * total_weight within
// rel 1e-9 / abs 1e-12.  Here one warp walks each row: the sortedness and
// weight tests are per arc, and with strictly increasing rows the lexsort
// equality is equivalent to "every arc (i, j, w) has a reverse (j, i, w)",
// found by binary search in row j.  Row weight sums are accumulated in
// binary64 (the identity is checked within the reference's tolerance, so the
// summation order does not matter).
#include "slpa_internal.cuh"

namespace {

constexpr int kVT = 256;

template <class W>
__global__ void __launch_bounds__(kVT) k_validate_rows(const int64_t *__restrict__ off, const int32_t *__restrict__ tgt,
                                                       const W *__restrict__ w, int64_t n,
                                                       unsigned long long *first_unsorted, unsigned *bad_weight,
                                                       unsigned *asym, double *sums) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double tot = 0.0, degsum = 0.0;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const int64_t lo = off[i], hi = off[i + 1];
        bool unsorted = false, badw = false, nosym = false;
        double rs = 0.0;
        for (int64_t e = lo + lane; e < hi; e += 32) {
            const int32_t j = tgt[e];
            const W x = w[e];
            rs += (double)x;
            if (e > lo && tgt[e - 1] >= j) unsorted = true;
            if (!(x > (W)0)) badw = true;
            // reverse arc (j, i) in row j, same weight
            int64_t a = off[j], b = off[j + 1];
            while (a < b) {
                const int64_t mid = (a + b) >> 1;
                if (tgt[mid] < i) a = mid + 1;
                else b = mid;
            }
            if (a >= off[j + 1] || tgt[a] != (int32_t)i || !(w[a] == x)) nosym = true;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
        degsum += rs;
        tot += rs;
        if (__any_sync(0xffffffffu, unsorted) && lane == 0) atomicMin(first_unsorted, (unsigned long long)i);
        if (__any_sync(0xffffffffu, badw) && lane == 0) atomicOr(bad_weight, 1u);
        if (__any_sync(0xffffffffu, nosym) && lane == 0) atomicOr(asym, 1u);
    }
    if (lane == 0) {
        atomicAdd(&sums[0], degsum);
        atomicAdd(&sums[1], tot);
    }
}

}  // namespace

// code: 0 ok, 1 unsorted (vertex), 2 non-positive weight, 3 asymmetric,
// 4 degree sum mismatch.  deg_sum / total: the two sides of the identity.
void slpa_validate_graph_impl(slpa_ctx *ctx, int32_t *code, int64_t *vertex, double *deg_sum, double *total) {
    DeviceGraph &g = ctx->g;
    const Csr &c = g.base;
    cudaStream_t s = ctx->stream;
    DevBuf<unsigned long long> buf;
    buf.alloc(6);
    unsigned long long init[6] = {~0ull, 0, 0, 0, 0, 0};
    CUDA_TRY(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
    unsigned *bw = reinterpret_cast<unsigned *>(buf.p + 1);
    unsigned *as = reinterpret_cast<unsigned *>(buf.p + 2);
    double *sums = reinterpret_cast<double *>(buf.p + 3);
    if (c.n > 0) {
        int dev_sms = 148;
        cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->device);
        const int64_t want = (c.n * 32 + kVT - 1) / kVT;
        const unsigned blocks = (unsigned)std::min<int64_t>(want, (int64_t)dev_sms * 8);
        if (g.w_f64)
            k_validate_rows<double><<<blocks, kVT, 0, s>>>(c.off.p, c.tgt.p, c.w64.p, c.n, buf.p, bw, as, sums);
        else
            k_validate_rows<float><<<blocks, kVT, 0, s>>>(c.off.p, c.tgt.p, c.w32.p, c.n, buf.p, bw, as, sums);
        CUDA_TRY(cudaGetLastError());
    }
    unsigned long long h[6];
    CUDA_TRY(cudaMemcpyAsync(h, buf.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    buf.release();
    double hs[2];
    memcpy(hs, &h[3], sizeof(hs));
    *deg_sum = hs[0];
    *total = hs[1];
    *vertex = -1;
    if (h[0] != ~0ull) {
        *code = 1;
        *vertex = (int64_t)h[0];
    } else if ((unsigned)h[1]) {
        *code = 2;
    } else if ((unsigned)h[2]) {
        *code = 3;
    } else {
        *code = 0;  // the degree-sum identity is judged by the caller (math.isclose)
    }
}
