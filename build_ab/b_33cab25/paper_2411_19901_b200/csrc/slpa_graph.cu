// slpa_graph.cu -- resident CSR management: validation (graph.py:55-68),
// symmetry detection + reverse CSR, visiting-order permutation (lpa.py:283-288),
// degree binning (lpa.py:137, :173), and device-side synthetic generators with
// canonical assembly (graph.py:107-139).  One-time setup work; the sweep
// kernels are in slpa_sweep.cu.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <vector>
#include <cub/cub.cuh>
#include "slpa_internal.cuh"

namespace {
constexpr int kT = 256;

// ------------------------------------------------------------------ validation
// err bits: 1 offsets[0] != 0, 2 decreasing offsets, 4 offsets[n] != m,
//           8 target out of range, 16 weight not > 0
__global__ void k_validate_offsets(const int64_t *off, int64_t n, int64_t m, unsigned *err) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    if (i == 0 && off[0] != 0) atomicOr(err, 1u);
    if (i < n && off[i + 1] < off[i]) atomicOr(err, 2u);
    if (i == n && off[n] != m) atomicOr(err, 4u);
}
template <class W>
__global__ void k_validate_arcs(const int32_t *tgt, const W *w, int64_t n, int64_t m, unsigned *err) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    int32_t t = tgt[i];
    if (t < 0 || t >= n) atomicOr(err, 8u);
    if (!(w[i] > (W)0)) atomicOr(err, 16u);
}

// ------------------------------------------------------------------ symmetry
// The arc multiset is symmetric iff sum_arcs h(u,t) == sum_arcs h(t,u) for a
// random-looking h; two independent 64-bit mixes make a false "symmetric"
// verdict a 2^-128 event.  One coalesced pass, one atomic per warp.
__device__ __forceinline__ uint64_t sym_mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
__global__ void k_sym_hash(const int64_t *off, const int32_t *tgt, int64_t n, unsigned long long *acc) {
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    uint64_t f1 = 0, r1 = 0, f2 = 0, r2 = 0;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
        const int64_t lo = off[v], hi = off[v + 1];
        for (int64_t e = lo + lane; e < hi; e += 32) {
            const uint64_t t = (uint64_t)(uint32_t)tgt[e], u = (uint64_t)v;
            const uint64_t fw = (u << 32) | t, rv = (t << 32) | u;
            f1 += sym_mix(fw);
            r1 += sym_mix(rv);
            f2 += sym_mix(fw ^ 0x5851F42D4C957F2DULL) * 0x2545F4914F6CDD1DULL;
            r2 += sym_mix(rv ^ 0x5851F42D4C957F2DULL) * 0x2545F4914F6CDD1DULL;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        f1 += __shfl_xor_sync(0xffffffffu, f1, o);
        r1 += __shfl_xor_sync(0xffffffffu, r1, o);
        f2 += __shfl_xor_sync(0xffffffffu, f2, o);
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    }
    if (lane == 0) {
        atomicAdd(&acc[0], (unsigned long long)f1);
        atomicAdd(&acc[1], (unsigned long long)r1);
        atomicAdd(&acc[2], (unsigned long long)f2);
        atomicAdd(&acc[3], (unsigned long long)r2);
    }
}

__global__ void k_in_degree(const int64_t *off, const int32_t *tgt, int64_t n, int64_t *indeg) {
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps)
        for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32)
            atomicAdd((unsigned long long *)&indeg[tgt[e]], 1ull);
}
__global__ void k_fill_reverse(const int64_t *off, const int32_t *tgt, int64_t n, int64_t *cursor, int32_t *rsrc) {
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps)
        for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
            unsigned long long p = atomicAdd((unsigned long long *)&cursor[tgt[e]], 1ull);
            rsrc[p] = (int32_t)v;
        }
}

// ------------------------------------------------------------------ integer precondition
// Every weight an integer >= 1 and every weighted degree < 2^31: then all
// sketch / vote values are integers < 2^31 and uint32 arithmetic reproduces
// the reference's binary64 arithmetic exactly.
template <class W>
__global__ void k_int_check(const int64_t *off, const W *w, int64_t n, unsigned *bad) {
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n; v += warps) {
        double sum = 0.0;
        bool ok = true;
        for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
            const double x = (double)w[e];
            ok &= (x >= 1.0) && (x == floor(x)) && (x < 2147483648.0);
            sum += x;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        ok = __all_sync(0xffffffffu, ok) && sum < 2147483648.0;
        if (!ok && lane == 0) atomicOr(bad, 1u);
    }
}

// ------------------------------------------------------------------ order
__global__ void k_order_scatter(const int64_t *order, int64_t n, int32_t *ids, int32_t *pos, unsigned *seen,
                                unsigned *err) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int64_t id = order[p];
    if (id < 0 || id >= n) {
        atomicOr(err, 1u);
        return;
    }
    ids[p] = (int32_t)id;
    pos[id] = (int32_t)p;
    if (atomicAdd(&seen[id], 1u) != 0) atomicOr(err, 1u);
}
__global__ void k_perm_degree(const int64_t *off, const int32_t *ids, int64_t n, int64_t *deg) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int32_t id = ids[p];
    deg[p] = off[id + 1] - off[id];
}
template <class W>
__global__ void k_perm_rows(const int64_t *off, const int32_t *tgt, const W *w, const int32_t *ids, const int32_t *pos,
                            const int64_t *poff, int32_t *ptgt, W *pw, int64_t n) {
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += warps) {
        const int32_t id = ids[p];
        const int64_t lo = off[id], hi = off[id + 1], dst = poff[p];
        for (int64_t e = lo + lane; e < hi; e += 32) {
            ptgt[dst + (e - lo)] = pos[tgt[e]];
            pw[dst + (e - lo)] = w[e];
        }
    }
}

// ------------------------------------------------------------------ bins
__global__ void k_classify(const int64_t *off, int64_t n, int32_t thr, int32_t hsplit, int32_t gsplit,
                           int32_t single, uint8_t *cls) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    int64_t d = off[v + 1] - off[v];
    cls[v] = d == 0 ? CLS_NONE
                    : ((single || d < thr) ? CLS_LO : (d < hsplit ? CLS_MID : (d < gsplit ? CLS_HI : CLS_GIANT)));
}
struct IsClass {
    const uint8_t *cls;
    uint8_t c;
    __host__ __device__ bool operator()(const int32_t &v) const { return cls[v] == c; }
};
__global__ void k_bin_degrees(const int64_t *off, const int32_t *bin, int64_t cnt, int64_t *deg) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) deg[i] = off[bin[i] + 1] - off[bin[i]];
}

// ------------------------------------------------------------------ generators
// Specification: DESIGN.md §6; CPU twin: oracle/lpa_oracle.c.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t h64(uint64_t seed, uint64_t ctr) { return splitmix64(splitmix64(seed) ^ ctr); }
__device__ __forceinline__ uint64_t perm_pow2(uint64_t x, int b, uint64_t key) {
    if (b == 0) return 0;
    uint64_t mask = (b >= 64) ? ~0ULL : ((1ULL << b) - 1);
    int sh = b / 2 + 1;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        uint64_t k = splitmix64(key + (uint64_t)r);
        x = (x * (k | 1ULL)) & mask;
        if (sh < b) x ^= x >> sh;
        x = (x + (k >> 17)) & mask;
    }
    return x;
}
__device__ __forceinline__ uint64_t perm_n(uint64_t x, uint64_t n, int b, uint64_t key) {
    uint64_t y = perm_pow2(x, b, key);
    while (y >= n) y = perm_pow2(y, b, key);
    return y;
}

// Edge keys: (min << 32 | max); dropped edges (self-loops) get `drop`.
__global__ void k_gen_rmat(int32_t scale, int64_t e0, int64_t count, uint32_t tA, uint32_t tAB, uint32_t tABC,
                           uint64_t seed, int32_t permute, uint64_t perm_key, uint64_t drop, uint64_t *keys) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int64_t e = e0 + i;
    const uint64_t W = (uint64_t)(scale + 1) / 2;
    uint64_t u = 0, v = 0, word = 0;
    for (int l = 0; l < scale; ++l) {
        if ((l & 1) == 0) word = h64(seed, (uint64_t)e * W + (uint64_t)(l >> 1));
        uint32_t r = (l & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
        uint64_t bit = 1ULL << (scale - 1 - l);
        if (r < tA) {
        } else if (r < tAB) v |= bit;
        else if (r < tABC) u |= bit;
        else { u |= bit; v |= bit; }
    }
    if (permute) {
        u = perm_pow2(u, scale, perm_key);
        v = perm_pow2(v, scale, perm_key);
    }
    if (u == v) { keys[i] = drop; return; }
    uint64_t a = u < v ? u : v, b = u < v ? v : u;
    keys[i] = (a << 32) | b;
}

__global__ void k_gen_grid(int64_t rows, int64_t cols, int32_t permute, uint64_t perm_key, int bits, uint64_t drop,
                           uint64_t *keys) {
    // edge index: 2 per cell (right, down)
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = rows * cols;
    if (i >= 2 * n) return;
    const int64_t cell = i >> 1;
    const int64_t r = cell / cols, c = cell % cols;
    uint64_t v = (uint64_t)cell, w;
    if ((i & 1) == 0) {
        if (c + 1 >= cols) { keys[i] = drop; return; }
        w = v + 1;
    } else {
        if (r + 1 >= rows) { keys[i] = drop; return; }
        w = v + (uint64_t)cols;
    }
    if (permute) {
        v = perm_n(v, (uint64_t)n, bits, perm_key);
        w = perm_n(w, (uint64_t)n, bits, perm_key);
    }
    uint64_t a = v < w ? v : w, b = v < w ? w : v;
    keys[i] = (a << 32) | b;
}

__global__ void k_gen_kmer(int64_t n, uint32_t keep, uint64_t seed, int32_t permute, uint64_t perm_key, int bits,
                           uint64_t drop, uint64_t *keys) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t chords = n / 20;
    if (i >= (n - 1) + chords) return;
    uint64_t a, b;
    if (i < n - 1) {
        uint64_t x = h64(seed, (uint64_t)i);
        if ((uint32_t)(x >> 32) >= keep) { keys[i] = drop; return; }
        a = (uint64_t)i;
        b = (uint64_t)i + 1;
    } else {
        int64_t c = i - (n - 1);
        uint64_t x = h64(seed ^ 0xC0DEULL, (uint64_t)c);
        a = (uint64_t)(uint32_t)x % (uint64_t)n;
        b = (x >> 32) % (uint64_t)n;
        if (a == b) { keys[i] = drop; return; }
    }
    if (permute) {
        a = perm_n(a, (uint64_t)n, bits, perm_key);
        b = perm_n(b, (uint64_t)n, bits, perm_key);
    }
    uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
    keys[i] = (lo << 32) | hi;
}

// unique pairs (a<=b, count) -> arc keys (src<<32|dst) with weights
// Arcs a->b and b->a of a unique pair, restricted to sources in [r0, r1)
// (the whole graph, or one rank's rows of a vertex-range partition).
__global__ void k_pair_arity(const uint64_t *pairs, int64_t np, int64_t *arity, int64_t r0, int64_t r1) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const uint64_t p = pairs[i];
    const int64_t a = (int64_t)(p >> 32), b = (int64_t)(p & 0xFFFFFFFFULL);
    arity[i] = (a >= r0 && a < r1) + (a != b && b >= r0 && b < r1);
}
template <class W>
__global__ void k_emit_arcs(const uint64_t *pairs, const double *wsum, const int64_t *pos, int64_t np, uint64_t *akeys,
                            W *aw, int64_t r0, int64_t r1) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const uint64_t p = pairs[i];
    const uint64_t a = p >> 32, b = p & 0xFFFFFFFFULL;
    int64_t o = pos[i];
    if ((int64_t)a >= r0 && (int64_t)a < r1) {
        akeys[o] = (a << 32) | b;
        aw[o] = (W)wsum[i];
        ++o;
    }
    if (a != b && (int64_t)b >= r0 && (int64_t)b < r1) {
        akeys[o] = (b << 32) | a;
        aw[o] = (W)wsum[i];
    }
}
__global__ void k_counts_to_double(const uint32_t *cnt, int64_t np, double *w) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < np) w[i] = (double)cnt[i];
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src),
// which np.add.reduceat applies to every segment after its first element.
__device__ __noinline__ double np_pairwise(const double *v, const int64_t *idx, int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; ++i) res += v[idx[i]];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = v[idx[j]];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += v[idx[i + j]];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += v[idx[i]];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise(v, idx, n2) + np_pairwise(v, idx + n2, n - n2);
}
// graph.py:127: pw = np.add.reduceat(w, starts) over the stably sorted entries
__global__ void k_run_sums(const double *w, const int64_t *idx, const int64_t *start, const uint32_t *cnt, int64_t np,
                           double *out) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= np) return;
    const int64_t s = start[r], c = cnt[r];
    double acc = w[idx[s]];
    if (c > 1) acc += np_pairwise(w, idx + s + 1, c - 1);
    out[r] = acc;
}
__global__ void k_pair_keys(const int64_t *src, const int64_t *dst, int64_t ne, uint64_t *keys, int64_t *idx) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ne) return;
    uint64_t a = (uint64_t)src[i], b = (uint64_t)dst[i];
    keys[i] = a < b ? ((a << 32) | b) : ((b << 32) | a);
    idx[i] = i;
}
// offsets[v] = lower_bound(akeys, v << 32)
__global__ void k_offsets_from_keys(const uint64_t *akeys, int64_t m, int64_t n, int64_t *off) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v > n) return;
    uint64_t key = (uint64_t)v << 32;
    int64_t a = 0, b = m;
    while (a < b) {
        int64_t mid = (a + b) >> 1;
        if (akeys[mid] < key) a = mid + 1;
        else b = mid;
    }
    off[v] = a;
}
__global__ void k_low32(const uint64_t *akeys, int64_t m, int32_t *tgt) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) tgt[i] = (int32_t)(akeys[i] & 0xFFFFFFFFULL);
}

int ceil_log2(uint64_t n) {
    int b = 0;
    while ((1ULL << b) < n) ++b;
    return b;
}

unsigned read_flag(slpa_ctx *ctx, unsigned *d) {
    unsigned h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return h;
}

template <class F>
void cub_call(slpa_ctx *ctx, F &&f) {
    size_t need = 0;
    CUDA_TRY(f((void *)nullptr, need));
    ctx->wb.scratch.alloc(need + 1);
    CUDA_TRY(f((void *)ctx->wb.scratch.p, need));
}

unsigned grid_warps(int64_t items) {
    int64_t b = (items * 32 + kT - 1) / kT;
    if (b > 148 * 64) b = 148 * 64;
    if (b < 1) b = 1;
    return (unsigned)b;
}
}  // namespace

// =====================================================================
void slpa_graph_validate(slpa_ctx *ctx, const Csr &c, int w_f64) {
    DevBuf<unsigned> err;
    err.alloc(1);
    CUDA_TRY(cudaMemsetAsync(err.p, 0, sizeof(unsigned), ctx->stream));
    k_validate_offsets<<<grid_for(c.n + 1, kT), kT, 0, ctx->stream>>>(c.off.p, c.n, c.m, err.p);
    if (c.m > 0) {
        if (w_f64)
            k_validate_arcs<double><<<grid_for(c.m, kT), kT, 0, ctx->stream>>>(c.tgt.p, c.w64.p, c.n, c.m, err.p);
        else
            k_validate_arcs<float><<<grid_for(c.m, kT), kT, 0, ctx->stream>>>(c.tgt.p, c.w32.p, c.n, c.m, err.p);
    }
    CUDA_TRY(cudaGetLastError());
    unsigned e = read_flag(ctx, err.p);
    err.release();
    if (e & 1) throw SlpaError{SLPA_EINVAL, "offsets must be a 1-d array starting at 0"};
    if (e & 2) throw SlpaError{SLPA_EINVAL, "offsets must be non-decreasing"};
    if (e & 4) throw SlpaError{SLPA_EINVAL, "offsets[-1] must equal the arc count"};
    if (e & 8) throw SlpaError{SLPA_EINVAL, "arc target out of range"};
    if (e & 16) throw SlpaError{SLPA_EINVAL, "arc weights must be positive"};
}

void slpa_check_int_weights(slpa_ctx *ctx) {
    DeviceGraph &g = ctx->g;
    cudaStream_t s = ctx->stream;
    g.int_weights = 1;
    if (g.n == 0 || g.m == 0) return;
    DevBuf<unsigned> bad;
    bad.alloc(1);
    CUDA_TRY(cudaMemsetAsync(bad.p, 0, sizeof(unsigned), s));
    if (g.w_f64)
        k_int_check<double><<<grid_warps(g.n), kT, 0, s>>>(g.off(), (const double *)g.w(), g.n, bad.p);
    else
        k_int_check<float><<<grid_warps(g.n), kT, 0, s>>>(g.off(), (const float *)g.w(), g.n, bad.p);
    CUDA_TRY(cudaGetLastError());
    g.int_weights = read_flag(ctx, bad.p) == 0;
    bad.release();
}

// ------------------------------------------------------------------ fused arc checks
// One arc-parallel pass: a block takes kArcBlock consecutive arcs, thread 0
// finds the rows they span, every thread locates the row of its first arc by
// a binary search inside that span and walks its kArcPer arcs.  Per arc: the
// symmetry multiset hashes of (u, t) and (t, u) (two independent 32-bit
// mixes summed in 64 bits), and the integral-weight test with the maximum
// weight; per row start: the maximum degree.  Replaces a warp-per-row pass
// whose hub rows serialised on one warp.
constexpr int kArcBlock = 2048, kArcPer = 8;

__device__ __forceinline__ uint32_t fmix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x85ebca6bu;
    x ^= x >> 13;
    x *= 0xc2b2ae35u;
    x ^= x >> 16;
    return x;
}
__device__ __forceinline__ int64_t row_of(const int64_t *off, int64_t lo, int64_t hi, int64_t e) {
    while (lo < hi) {  // largest r in [lo, hi] with off[r] <= e
        const int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(&off[mid]) <= e) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

template <class W>
__global__ void __launch_bounds__(256) k_arc_checks(const int64_t *off, const int32_t *tgt, const W *w, int64_t n,
                                                    int64_t m, unsigned long long *acc, unsigned *bad,
                                                    unsigned long long *wmax, unsigned long long *dmax,
                                                    int64_t e_begin = 0) {
    // arcs [e_begin, m) -- the whole graph, or one chunk of a pipelined upload
    __shared__ int64_t s_r[2];
    const int64_t e0 = e_begin + (int64_t)blockIdx.x * kArcBlock;
    if (e0 >= m) return;
    const int64_t e1 = min(m, e0 + kArcBlock);
    if (threadIdx.x == 0) {
        s_r[0] = row_of(off, 0, n - 1, e0);
        s_r[1] = row_of(off, s_r[0], n - 1, e1 - 1);
    }
    __syncthreads();
    unsigned long long f1 = 0, r1 = 0, f2 = 0, r2 = 0, mw = 0, md = 0;
    bool ok = true;
    const int64_t a0 = e0 + (int64_t)threadIdx.x * kArcPer;
    if (a0 < e1) {
        int64_t u = row_of(off, s_r[0], s_r[1], a0);
        int64_t start = __ldg(&off[u]), next = __ldg(&off[u + 1]);
        uint32_t hu1 = fmix32((uint32_t)u ^ 0x9e3779b9u), hu2 = fmix32((uint32_t)u ^ 0x7f4a7c15u);
        if (start >= a0) md = (unsigned long long)(next - start);
        for (int j = 0; j < kArcPer; ++j) {
            const int64_t e = a0 + j;
            if (e >= e1) break;
            while (e >= next && u < n - 1) {  // (bounded: offsets are validated concurrently)
                ++u;
                start = next;
                next = __ldg(&off[u + 1]);
                hu1 = fmix32((uint32_t)u ^ 0x9e3779b9u);
                hu2 = fmix32((uint32_t)u ^ 0x7f4a7c15u);
                const unsigned long long d = (unsigned long long)(next - start);
                md = d > md ? d : md;
            }
            const uint32_t t = (uint32_t)__ldg(&tgt[e]);
            const uint32_t ht1 = fmix32(t ^ 0x9e3779b9u), ht2 = fmix32(t ^ 0x7f4a7c15u);
            f1 += fmix32(hu1 + t);
            r1 += fmix32(ht1 + (uint32_t)u);
            f2 += fmix32(hu2 ^ (t * 0x2545f491u));
            r2 += fmix32(ht2 ^ ((uint32_t)u * 0x2545f491u));
            const double x = (double)__ldg(&w[e]);
            ok &= (x >= 1.0) && (x == floor(x)) && (x < 2147483648.0);
            const unsigned long long xi = ok ? (unsigned long long)x : 0ull;
            mw = xi > mw ? xi : mw;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        f1 += __shfl_xor_sync(0xffffffffu, f1, o);
        r1 += __shfl_xor_sync(0xffffffffu, r1, o);
        f2 += __shfl_xor_sync(0xffffffffu, f2, o);
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
        const unsigned long long ow = __shfl_xor_sync(0xffffffffu, mw, o), od = __shfl_xor_sync(0xffffffffu, md, o);
        mw = ow > mw ? ow : mw;
        md = od > md ? od : md;
    }
    ok = __all_sync(0xffffffffu, ok);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&acc[0], f1);
        atomicAdd(&acc[1], r1);
        atomicAdd(&acc[2], f2);
        atomicAdd(&acc[3], r2);
        atomicMax(wmax, mw);
        atomicMax(dmax, md);
        if (!ok) atomicOr(bad, 1u);
    }
}

// The four symmetry hash sums of k_arc_checks over the resident rows (a
// partition's rows: the sums add up across ranks; the graph is symmetric iff
// the forward and reverse sums agree globally).
void slpa_arc_hash_impl(slpa_ctx *ctx, uint64_t out[4]) {
    DeviceGraph &g = ctx->g;
    cudaStream_t s = ctx->stream;
    for (int i = 0; i < 4; ++i) out[i] = 0;
    if (g.n == 0 || g.m == 0) return;
    DevBuf<unsigned long long> acc;
    acc.alloc(8);
    CUDA_TRY(cudaMemsetAsync(acc.p, 0, 8 * sizeof(unsigned long long), s));
    const unsigned blocks = (unsigned)((g.m + kArcBlock - 1) / kArcBlock);
    if (g.w_f64)
        k_arc_checks<double><<<blocks, 256, 0, s>>>(g.off(), g.tgt(), (const double *)g.w(), g.n, g.m, acc.p,
                                                      (unsigned *)(acc.p + 4), acc.p + 5, acc.p + 6);
    else
        k_arc_checks<float><<<blocks, 256, 0, s>>>(g.off(), g.tgt(), (const float *)g.w(), g.n, g.m, acc.p,
                                                     (unsigned *)(acc.p + 4), acc.p + 5, acc.p + 6);
    CUDA_TRY(cudaGetLastError());
    unsigned long long h[8];
    CUDA_TRY(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int i = 0; i < 4; ++i) out[i] = h[i];
}

// k_arc_checks over arcs [e0, e1) of `c` into acc[0..7] (stream order).
void slpa_arc_checks_range(slpa_ctx *ctx, const Csr &c, int w_f64, int64_t e0, int64_t e1, unsigned long long *acc) {
    if (e1 <= e0) return;
    const unsigned blocks = (unsigned)((e1 - e0 + kArcBlock - 1) / kArcBlock);
    cudaStream_t s = ctx->stream;
    if (w_f64)
        k_arc_checks<double><<<blocks, 256, 0, s>>>(c.off.p, c.tgt.p, c.w64.p, c.n, e1, acc, (unsigned *)(acc + 4),
                                                      acc + 5, acc + 6, e0);
    else
        k_arc_checks<float><<<blocks, 256, 0, s>>>(c.off.p, c.tgt.p, c.w32.p, c.n, e1, acc, (unsigned *)(acc + 4),
                                                     acc + 5, acc + 6, e0);
    CUDA_TRY(cudaGetLastError());
}

// k_validate_arcs over arcs [e0, e1) (stream order; flags into err).
void slpa_validate_arcs_range(slpa_ctx *ctx, const Csr &c, int w_f64, int64_t e0, int64_t e1, unsigned *err) {
    if (e1 <= e0) return;
    if (w_f64)
        k_validate_arcs<double><<<grid_for(e1 - e0, kT), kT, 0, ctx->stream>>>(c.tgt.p + e0, c.w64.p + e0, c.n,
                                                                                e1 - e0, err);
    else
        k_validate_arcs<float><<<grid_for(e1 - e0, kT), kT, 0, ctx->stream>>>(c.tgt.p + e0, c.w32.p + e0, c.n,
                                                                               e1 - e0, err);
    CUDA_TRY(cudaGetLastError());
}

// Offsets check of a freshly copied CSR (flags into err; stream order).
void slpa_validate_offsets_async(slpa_ctx *ctx, const Csr &c, unsigned *err) {
    k_validate_offsets<<<grid_for(c.n + 1, kT), kT, 0, ctx->stream>>>(c.off.p, c.n, c.m, err);
    CUDA_TRY(cudaGetLastError());
}

void slpa_throw_validation(unsigned e) {
    if (e & 1) throw SlpaError{SLPA_EINVAL, "offsets must be a 1-d array starting at 0"};
    if (e & 2) throw SlpaError{SLPA_EINVAL, "offsets must be non-decreasing"};
    if (e & 4) throw SlpaError{SLPA_EINVAL, "offsets[-1] must equal the arc count"};
    if (e & 8) throw SlpaError{SLPA_EINVAL, "arc target out of range"};
    if (e & 16) throw SlpaError{SLPA_EINVAL, "arc weights must be positive"};
}

// Symmetry check + reverse CSR of the active numbering; resets the bins.
void slpa_graph_finalize(slpa_ctx *ctx) {
    DeviceGraph &g = ctx->g;
    cudaStream_t s = ctx->stream;
    g.max_deg = -1;
    g.bin_thr = -1;
    g.bin_single = -1;
    g.bin_lo_sorted = -1;
    g.roff.release();
    g.rsrc.release();
    g.symmetric = 1;
    g.int_weights = 1;
    const bool pre = ctx->pre_checks_valid;
    ctx->pre_checks_valid = 0;
    if (g.n == 0 || g.m == 0) return;
    // acc: 4 hashes, bad flag, max weight, max degree (one readback); a
    // pipelined upload computed them while the arcs were copied
    unsigned long long h[8];
    if (pre) {
        for (int i = 0; i < 8; ++i) h[i] = ctx->pre_checks[i];
    } else {
        DevBuf<unsigned long long> acc;
        acc.alloc(8);
        CUDA_TRY(cudaMemsetAsync(acc.p, 0, 8 * sizeof(unsigned long long), s));
        slpa_arc_checks_range(ctx, g.act(), g.w_f64, 0, g.m, acc.p);
        CUDA_TRY(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    g.symmetric = (h[0] == h[1]) && (h[2] == h[3]);
    g.max_deg = (int64_t)h[6];
    // integer sketch values need integral weights and every weighted degree
    // < 2^31: max weight x max degree < 2^31 settles it; otherwise the exact
    // per-row sums decide
    if ((unsigned)h[4] != 0u) g.int_weights = 0;
    else if ((double)h[5] * (double)h[6] >= 2147483648.0) slpa_check_int_weights(ctx);
    if (g.symmetric) return;
    // reverse CSR: in-degree histogram, exclusive scan, atomic fill
    g.roff.alloc(g.n + 1);
    g.rsrc.alloc(g.m);
    DevBuf<int64_t> cursor;
    cursor.alloc(g.n + 1);
    CUDA_TRY(cudaMemsetAsync(cursor.p, 0, (g.n + 1) * sizeof(int64_t), s));
    k_in_degree<<<grid_warps(g.n), kT, 0, s>>>(g.off(), g.tgt(), g.n, cursor.p);
    int64_t *in = cursor.p, *out = g.roff.p;
    int64_t nn = g.n + 1;
    cub_call(ctx, [&](void *tmp, size_t &bytes) {
        return cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, nn, s);
    });
    CUDA_TRY(cudaMemcpyAsync(cursor.p, g.roff.p, (g.n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    k_fill_reverse<<<grid_warps(g.n), kT, 0, s>>>(g.off(), g.tgt(), g.n, cursor.p, g.rsrc.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));
    cursor.release();
}

// Visiting order (lpa.py:283-288): order[p] = vertex visited p-th.
void slpa_graph_apply_order(slpa_ctx *ctx, const int64_t *order, bool on_device) {
    DeviceGraph &g = ctx->g;
    cudaStream_t s = ctx->stream;
    g.perm.release();
    g.ids.release();
    g.pos.release();
    g.has_order = 0;
    if (!order) {
        slpa_graph_finalize(ctx);
        return;
    }
    ctx->pre_checks_valid = 0;  // the checks run on the permuted CSR (the reverse CSR must be built in it)
    const int64_t n = g.n, m = g.m;
    DevBuf<int64_t> d_order;
    const int64_t *ord = order;
    if (!on_device) {
        d_order.alloc(n);
        CUDA_TRY(cudaMemcpyAsync(d_order.p, order, n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        ord = d_order.p;
    }
    g.ids.alloc(n);
    g.pos.alloc(n);
    DevBuf<unsigned> seen, err;
    seen.alloc(n);
    err.alloc(1);
    CUDA_TRY(cudaMemsetAsync(seen.p, 0, n * sizeof(unsigned), s));
    CUDA_TRY(cudaMemsetAsync(err.p, 0, sizeof(unsigned), s));
    if (n > 0) k_order_scatter<<<grid_for(n, kT), kT, 0, s>>>(ord, n, g.ids.p, g.pos.p, seen.p, err.p);
    CUDA_TRY(cudaGetLastError());
    if (read_flag(ctx, err.p)) {
        g.ids.release();
        g.pos.release();
        throw SlpaError{SLPA_EINVAL, "order must be a permutation of all vertex ids"};
    }
    seen.release();
    err.release();
    d_order.release();
    // permuted CSR
    g.perm.n = n;
    g.perm.m = m;
    g.perm.off.alloc(n + 1);
    g.perm.tgt.alloc(m);
    if (g.w_f64) g.perm.w64.alloc(m);
    else g.perm.w32.alloc(m);
    DevBuf<int64_t> deg;
    deg.alloc(n + 1);
    CUDA_TRY(cudaMemsetAsync(deg.p, 0, (n + 1) * sizeof(int64_t), s));
    if (n > 0) k_perm_degree<<<grid_for(n, kT), kT, 0, s>>>(g.base.off.p, g.ids.p, n, deg.p);
    int64_t *din = deg.p, *dout = g.perm.off.p;
    int64_t nn = n + 1;
    cub_call(ctx, [&](void *tmp, size_t &bytes) { return cub::DeviceScan::ExclusiveSum(tmp, bytes, din, dout, nn, s); });
    if (n > 0) {
        if (g.w_f64)
            k_perm_rows<double><<<grid_warps(n), kT, 0, s>>>(g.base.off.p, g.base.tgt.p, g.base.w64.p, g.ids.p, g.pos.p,
                                                             g.perm.off.p, g.perm.tgt.p, g.perm.w64.p, n);
        else
            k_perm_rows<float><<<grid_warps(n), kT, 0, s>>>(g.base.off.p, g.base.tgt.p, g.base.w32.p, g.ids.p, g.pos.p,
                                                            g.perm.off.p, g.perm.tgt.p, g.perm.w32.p, n);
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));
    deg.release();
    g.has_order = 1;
    slpa_graph_finalize(ctx);
}

static int64_t giant_split() {
    static int64_t v = [] {
        const char *e = getenv("SLPA_GIANT");
        return e ? std::max<int64_t>(1, atoll(e)) : (int64_t)32768;
    }();
    return v;
}

static int64_t hi_split() {
    static int64_t v = [] {
        const char *e = getenv("SLPA_HI_SPLIT");
        return e ? std::max<int64_t>(1, atoll(e)) : (int64_t)1;
    }();
    return v;
}

// Degree bins for a threshold (lpa.py:137, :173): low = 0 < deg < thr
// (ascending position), high = deg >= thr (descending degree, so the longest
// scans start first).  `single` puts every non-empty vertex in the low bin.
void slpa_ensure_bins(slpa_ctx *ctx, const slpa_config *cfg) {
    DeviceGraph &g = ctx->g;
    cudaStream_t s = ctx->stream;
    const int single = (cfg->variant == SLPA_VARIANT_EXACT) || (cfg->variant == SLPA_VARIANT_MG && cfg->shared_sketch) ||
                       slpa_large_k(cfg);
    // deterministic mode: degree-sorted low bin (homogeneous warps); async
    // mode: ascending positions (closest to the sequential visiting order,
    // which async quality depends on)
    static const int lo_sort_env = [] {
        const char *e = getenv("SLPA_LO_SORT");
        return e ? atoi(e) : -1;
    }();
    const int lo_sorted = lo_sort_env >= 0 ? lo_sort_env : (cfg->worker_count == 0);
    if (g.bin_thr == cfg->degree_threshold && g.bin_single == single && g.bin_lo_sorted == lo_sorted) return;
    const int64_t n = g.n;
    g.cls.alloc(n);
    g.bin_lo.alloc(n);
    g.bin_mid.alloc(n);
    g.bin_hi.alloc(n);
    // Bins are an execution split: lo = deg < D_H (one lane, one sketch),
    // mid = D_H <= deg < max(D_H, hi_split) (one lane, R_H chunks),
    // hi = the rest (one warp, lane = chunk).
    const int64_t hs = std::max<int64_t>(cfg->degree_threshold, hi_split());
    const int64_t gs = std::max<int64_t>(hs, giant_split());
    const int32_t hsplit = (int32_t)std::min<int64_t>(hs, INT32_MAX);
    const int32_t gsplit = (int32_t)std::min<int64_t>(gs, INT32_MAX);
    g.bin_giant.alloc(n);
    if (n > 0)
        k_classify<<<grid_for(n, kT), kT, 0, s>>>(g.off(), n, cfg->degree_threshold, hsplit, gsplit, single, g.cls.p);
    CUDA_TRY(cudaGetLastError());
    DevBuf<int64_t> &cnt = g.sort_small;  // persistent scratch: bins are rebuilt on every upload
    cnt.alloc(8);
    cub::CountingInputIterator<int32_t> it(0);
    const uint8_t classes[4] = {CLS_LO, CLS_MID, CLS_HI, CLS_GIANT};
    int32_t *outs[4] = {g.bin_lo.p, g.bin_mid.p, g.bin_hi.p, g.bin_giant.p};
    for (int which = 0; which < 4; ++which) {
        IsClass pred{g.cls.p, classes[which]};
        int32_t *out = outs[which];
        int64_t *nsel = cnt.p + which;
        cub_call(ctx, [&](void *tmp, size_t &bytes) {
            return cub::DeviceSelect::If(tmp, bytes, it, out, nsel, n, pred, s);
        });
    }
    int64_t h[4] = {0, 0, 0, 0};
    CUDA_TRY(cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    g.n_lo = h[0];
    g.n_mid = h[1];
    g.n_hi = h[2];
    g.n_giant = h[3];
    // hi / giant: descending degree (longest scans first); lo / mid:
    // ascending degree, stable on position (degree-homogeneous warps)
    for (int which = 0; which < 4; ++which) {
        const int64_t cntb = which >= 2 ? (which == 2 ? g.n_hi : g.n_giant)
                                        : (which == 1 ? g.n_mid : (lo_sorted ? g.n_lo : 0));
        int32_t *binp = outs[which];
        if (cntb <= 1) continue;
        DevBuf<int64_t> &dk = g.sort_k1, &dk2 = g.sort_k2;
        DevBuf<int32_t> &v2 = g.sort_v;
        dk.alloc(cntb);
        dk2.alloc(cntb);
        v2.alloc(cntb);
        k_bin_degrees<<<grid_for(cntb, kT), kT, 0, s>>>(g.off(), binp, cntb, dk.p);
        int64_t *k1 = dk.p, *k2 = dk2.p;
        int32_t *v1 = binp, *vv2 = v2.p;
        const int64_t nh = cntb;
        // degree keys: low / mid bins are bounded by their split, so few radix passes
        const int64_t kmax = (which == 0 && !single) ? (int64_t)cfg->degree_threshold
                                                     : (which == 1 ? (int64_t)hsplit : (1LL << 40));
        int end_bit = 1;
        while (end_bit < 40 && (1LL << end_bit) <= kmax) ++end_bit;
        if (which >= 2)
            cub_call(ctx, [&](void *tmp, size_t &bytes) {
                return cub::DeviceRadixSort::SortPairsDescending(tmp, bytes, k1, k2, v1, vv2, nh, 0, end_bit, s);
            });
        else
            cub_call(ctx, [&](void *tmp, size_t &bytes) {
                return cub::DeviceRadixSort::SortPairs(tmp, bytes, k1, k2, v1, vv2, nh, 0, end_bit, s);
            });
        CUDA_TRY(cudaMemcpyAsync(binp, v2.p, nh * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    }
    // largest light degree (the low bin is degree-ascending when sorted)
    g.lo_max_deg = single ? INT64_MAX : (int64_t)cfg->degree_threshold - 1;
    if (g.n_lo > 0 && lo_sorted && !single) {
        int32_t vlast = 0;
        CUDA_TRY(cudaMemcpyAsync(&vlast, g.bin_lo.p + g.n_lo - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        int64_t o2[2] = {0, 0};
        CUDA_TRY(cudaMemcpyAsync(o2, g.off() + vlast, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        g.lo_max_deg = o2[1] - o2[0];
    }
    // giant gather-buffer offsets: exclusive prefix of the giants' degrees
    g.giant_off.alloc(g.n_giant + 1);
    g.giant_arcs = 0;
    g.giant_max_deg = 0;
    if (g.n_giant > 0) {
        DevBuf<int64_t> &dk = g.sort_k1;
        dk.alloc(g.n_giant + 1);
        CUDA_TRY(cudaMemsetAsync(dk.p, 0, (g.n_giant + 1) * sizeof(int64_t), s));
        k_bin_degrees<<<grid_for(g.n_giant, kT), kT, 0, s>>>(g.off(), g.bin_giant.p, g.n_giant, dk.p);
        int64_t *din = dk.p, *dout = g.giant_off.p;
        const int64_t nn = g.n_giant + 1;
        cub_call(ctx, [&](void *tmp, size_t &bytes) { return cub::DeviceScan::ExclusiveSum(tmp, bytes, din, dout, nn, s); });
        CUDA_TRY(cudaMemcpyAsync(&g.giant_arcs, g.giant_off.p + g.n_giant, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        int64_t first2[2] = {0, 0};  // bin_giant is degree-descending: slot 0 is the largest
        CUDA_TRY(cudaMemcpyAsync(first2, g.giant_off.p, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        g.giant_max_deg = first2[1] - first2[0];
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    g.bin_thr = cfg->degree_threshold;
    g.bin_single = single;
    g.bin_lo_sorted = lo_sorted;
}

// Unique canonical pairs (a<=b, sorted) + merged float64 weights -> CSR:
// emit both arc directions (self-loop once, graph.py:131-134), sort arcs by
// (src, dst) (graph.py:135-136), offsets by binary search, cast weights.
template <class W>
static void assemble_pairs_t(slpa_ctx *ctx, int64_t n, DevBuf<uint64_t> &pairs, int64_t np, DevBuf<double> &wsum,
                             int end_bit, DevBuf<W> &out_w, int64_t r0, int64_t r1) {
    cudaStream_t s = ctx->stream;
    DeviceGraph &g = ctx->g;
    DevBuf<int64_t> arity, posn;
    arity.alloc(np + 1);
    posn.alloc(np + 1);
    CUDA_TRY(cudaMemsetAsync(arity.p, 0, (np + 1) * sizeof(int64_t), s));
    if (np > 0) k_pair_arity<<<grid_for(np, kT), kT, 0, s>>>(pairs.p, np, arity.p, r0, r1);
    {
        int64_t *ain = arity.p, *aout = posn.p;
        int64_t nn = np + 1;
        cub_call(ctx, [&](void *tmp, size_t &bytes) { return cub::DeviceScan::ExclusiveSum(tmp, bytes, ain, aout, nn, s); });
    }
    int64_t m = 0;
    CUDA_TRY(cudaMemcpyAsync(&m, posn.p + np, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    arity.release();
    DevBuf<uint64_t> akeys, akeys2;
    DevBuf<W> aw;
    akeys.alloc(m);
    aw.alloc(m);
    if (np > 0) k_emit_arcs<W><<<grid_for(np, kT), kT, 0, s>>>(pairs.p, wsum.p, posn.p, np, akeys.p, aw.p, r0, r1);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));
    pairs.release();
    wsum.release();
    posn.release();
    akeys2.alloc(m);
    out_w.alloc(m);
    {
        uint64_t *k1 = akeys.p, *k2 = akeys2.p;
        W *v1 = aw.p, *v2 = out_w.p;
        cub_call(ctx, [&](void *tmp, size_t &bytes) {
            return cub::DeviceRadixSort::SortPairs(tmp, bytes, k1, k2, v1, v2, m, 0, end_bit, s);
        });
    }
    akeys.release();
    aw.release();
    g.base.n = n;
    g.base.m = m;
    g.base.off.alloc(n + 1);
    g.base.tgt.alloc(m);
    k_offsets_from_keys<<<grid_for(n + 1, kT), kT, 0, s>>>(akeys2.p, m, n, g.base.off.p);
    if (m > 0) k_low32<<<grid_for(m, kT), kT, 0, s>>>(akeys2.p, m, g.base.tgt.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));
    akeys2.release();
    g.n = n;
    g.m = m;
    g.perm.release();
    g.ids.release();
    g.pos.release();
    g.has_order = 0;
    ctx->wb.scratch.release();
}

static void assemble_pairs(slpa_ctx *ctx, int64_t n, DevBuf<uint64_t> &pairs, int64_t np, DevBuf<double> &wsum,
                           int end_bit, int w_f64, int64_t r0 = 0, int64_t r1 = -1) {
    ctx->g.base.release();
    ctx->g.w_f64 = w_f64 ? 1 : 0;
    if (r1 < 0) r1 = n;
    if (w_f64) assemble_pairs_t<double>(ctx, n, pairs, np, wsum, end_bit, ctx->g.base.w64, r0, r1);
    else assemble_pairs_t<float>(ctx, n, pairs, np, wsum, end_bit, ctx->g.base.w32, r0, r1);
}

// Unit-weight edge keys (min<<32|max, `drop` = removed): sort, run-length
// encode (duplicate count = merged weight, exact in any order), assemble.
static void assemble_from_keys(slpa_ctx *ctx, int64_t n, DevBuf<uint64_t> &keys, int64_t ne, int end_bit,
                               int64_t r0 = 0, int64_t r1 = -1) {
    cudaStream_t s = ctx->stream;
    DevBuf<uint64_t> sorted;
    sorted.alloc(ne);
    {
        uint64_t *kin = keys.p, *kout = sorted.p;
        cub_call(ctx, [&](void *tmp, size_t &bytes) {
            return cub::DeviceRadixSort::SortKeys(tmp, bytes, kin, kout, ne, 0, end_bit, s);
        });
    }
    DevBuf<uint32_t> counts;
    DevBuf<int64_t> nruns;
    counts.alloc(ne);
    nruns.alloc(1);
    {
        uint64_t *kin = sorted.p, *uniq = keys.p;
        uint32_t *cnt = counts.p;
        int64_t *nr = nruns.p;
        cub_call(ctx, [&](void *tmp, size_t &bytes) {
            return cub::DeviceRunLengthEncode::Encode(tmp, bytes, kin, uniq, cnt, nr, ne, s);
        });
    }
    int64_t np = 0;
    CUDA_TRY(cudaMemcpyAsync(&np, nruns.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (np > 0) {  // the drop sentinel sorts last
        uint64_t last = 0;
        CUDA_TRY(cudaMemcpyAsync(&last, keys.p + np - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if ((last >> 32) >= (uint64_t)n) --np;
    }
    sorted.release();
    DevBuf<double> wsum;
    wsum.alloc(np);
    if (np > 0) k_counts_to_double<<<grid_for(np, kT), kT, 0, s>>>(counts.p, np, wsum.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));
    counts.release();
    assemble_pairs(ctx, n, keys, np, wsum, end_bit, 0, r0, r1);
}

static int key_end_bit(int64_t n) { return 32 + ceil_log2((uint64_t)(n > 1 ? n : 2)) + 1; }
static uint64_t drop_key(int64_t n) { return 1ULL << (key_end_bit(n) - 1); }

void slpa_gen_rmat_impl(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB, uint32_t tABC,
                        uint64_t seed, int32_t permute, uint64_t perm_key) {
    SLPA_REQUIRE(scale >= 1 && scale <= 31, SLPA_EINVAL, "rmat scale must be in [1, 31]");
    SLPA_REQUIRE(num_edges >= 0, SLPA_EINVAL, "num_edges must be non-negative");
    const int64_t n = 1LL << scale;
    DevBuf<uint64_t> keys;
    keys.alloc(num_edges);
    if (num_edges > 0)
        k_gen_rmat<<<grid_for(num_edges, kT), kT, 0, ctx->stream>>>(scale, 0, num_edges, tA, tAB, tABC, seed, permute,
                                                                    perm_key, drop_key(n), keys.p);
    CUDA_TRY(cudaGetLastError());
    assemble_from_keys(ctx, n, keys, num_edges, key_end_bit(n));
}

void slpa_gen_grid_impl(slpa_ctx *ctx, int64_t rows, int64_t cols, int32_t permute, uint64_t perm_key) {
    SLPA_REQUIRE(rows >= 1 && cols >= 1 && rows * cols < (1LL << 31), SLPA_EINVAL, "bad grid shape");
    const int64_t n = rows * cols;
    DevBuf<uint64_t> keys;
    keys.alloc(2 * n);
    k_gen_grid<<<grid_for(2 * n, kT), kT, 0, ctx->stream>>>(rows, cols, permute, perm_key, ceil_log2((uint64_t)n),
                                                             drop_key(n), keys.p);
    CUDA_TRY(cudaGetLastError());
    assemble_from_keys(ctx, n, keys, 2 * n, key_end_bit(n));
}

void slpa_gen_kmer_impl(slpa_ctx *ctx, int64_t n, uint32_t keep, uint64_t seed, int32_t permute, uint64_t perm_key) {
    SLPA_REQUIRE(n >= 2 && n < (1LL << 31), SLPA_EINVAL, "bad k-mer graph size");
    const int64_t ne = (n - 1) + n / 20;
    DevBuf<uint64_t> keys;
    keys.alloc(ne);
    k_gen_kmer<<<grid_for(ne, kT), kT, 0, ctx->stream>>>(n, keep, seed, permute, perm_key, ceil_log2((uint64_t)n),
                                                          drop_key(n), keys.p);
    CUDA_TRY(cudaGetLastError());
    assemble_from_keys(ctx, n, keys, ne, key_end_bit(n));
}

// build_graph (graph.py:142-162) on the device: canonical pairs, stable sort,
// float64 duplicate sums in reduceat order, both directions, sorted rows.
void slpa_build_graph_impl(slpa_ctx *ctx, int64_t n, int64_t ne, const int64_t *src, const int64_t *dst,
                           const double *w, int32_t weights_f64) {
    SLPA_REQUIRE(n >= 0 && n < (1LL << 31) - 1 && ne >= 0, SLPA_EINVAL, "bad graph size");
    for (int64_t i = 0; i < ne; ++i) {
        SLPA_REQUIRE(src[i] >= 0 && src[i] < n && dst[i] >= 0 && dst[i] < n, SLPA_EINVAL, "edge out of range");
        if (w) SLPA_REQUIRE(w[i] > 0 && std::isfinite(w[i]), SLPA_EINVAL, "edge must have a positive finite weight");
    }
    cudaStream_t s = ctx->stream;
    const int end_bit = key_end_bit(n);
    DevBuf<int64_t> d_src, d_dst, idx, idx2;
    DevBuf<uint64_t> keys, keys2;
    DevBuf<double> d_w;
    d_src.alloc(ne);
    d_dst.alloc(ne);
    d_w.alloc(ne);
    keys.alloc(ne);
    keys2.alloc(ne);
    idx.alloc(ne);
    idx2.alloc(ne);
    if (ne > 0) {
        CUDA_TRY(cudaMemcpyAsync(d_src.p, src, ne * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(d_dst.p, dst, ne * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        if (w) {
            CUDA_TRY(cudaMemcpyAsync(d_w.p, w, ne * sizeof(double), cudaMemcpyHostToDevice, s));
        } else {
            std::vector<double> ones((size_t)ne, 1.0);
            CUDA_TRY(cudaMemcpyAsync(d_w.p, ones.data(), ne * sizeof(double), cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaStreamSynchronize(s));
        }
        k_pair_keys<<<grid_for(ne, kT), kT, 0, s>>>(d_src.p, d_dst.p, ne, keys.p, idx.p);
        CUDA_TRY(cudaGetLastError());
        uint64_t *k1 = keys.p, *k2 = keys2.p;
        int64_t *v1 = idx.p, *v2 = idx2.p;
        cub_call(ctx, [&](void *tmp, size_t &bytes) {  // stable, like np.lexsort
            return cub::DeviceRadixSort::SortPairs(tmp, bytes, k1, k2, v1, v2, ne, 0, end_bit, s);
        });
    }
    d_src.release();
    d_dst.release();
    DevBuf<uint32_t> counts;
    DevBuf<int64_t> nruns, starts;
    counts.alloc(ne);
    nruns.alloc(1);
    CUDA_TRY(cudaMemsetAsync(nruns.p, 0, sizeof(int64_t), s));
    if (ne > 0) {
        uint64_t *kin = keys2.p, *uniq = keys.p;
        uint32_t *cnt = counts.p;
        int64_t *nr = nruns.p;
        cub_call(ctx, [&](void *tmp, size_t &bytes) {
            return cub::DeviceRunLengthEncode::Encode(tmp, bytes, kin, uniq, cnt, nr, ne, s);
        });
    }
    int64_t np = 0;
    CUDA_TRY(cudaMemcpyAsync(&np, nruns.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    starts.alloc(np + 1);
    DevBuf<double> wsum;
    wsum.alloc(np);
    if (np > 0) {
        DevBuf<int64_t> c64;
        c64.alloc(np);
        // exclusive scan of run lengths -> run starts
        uint32_t *cin = counts.p;
        int64_t *sout = starts.p;
        int64_t nn = np;
        cub_call(ctx, [&](void *tmp, size_t &bytes) { return cub::DeviceScan::ExclusiveSum(tmp, bytes, cin, sout, nn, s); });
        k_run_sums<<<grid_for(np, kT), kT, 0, s>>>(d_w.p, idx2.p, starts.p, counts.p, np, wsum.p);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    keys2.release();
    idx.release();
    idx2.release();
    d_w.release();
    counts.release();
    starts.release();
    assemble_pairs(ctx, n, keys, np, wsum, end_bit, weights_f64);
}

// ---------------------------------------------------------------- partition
namespace {
struct TouchesRange {
    int64_t r0, r1;
    __host__ __device__ bool operator()(const uint64_t &k) const {
        const int64_t a = (int64_t)(k >> 32), b = (int64_t)(k & 0xFFFFFFFFULL);
        return (a >= r0 && a < r1) || (b >= r0 && b < r1);
    }
};
}  // namespace

// Arc-balanced partition of the RMAT graph (multi-GPU): the
// same counter-based edge stream every rank generates, histogrammed by
// endpoint (self-loops dropped; duplicates counted, which the cut does not
// need to resolve), then world-1 cuts where the running arc count crosses
// r * total / world.  Every rank computes the same cuts.
__global__ void k_key_degrees(const uint64_t *__restrict__ keys, int64_t cnt, uint64_t drop,
                              unsigned long long *__restrict__ deg) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const uint64_t k = keys[i];
    if (k == drop) return;
    atomicAdd(&deg[k >> 32], 1ull);
    atomicAdd(&deg[k & 0xFFFFFFFFULL], 1ull);
}
__global__ void k_find_cuts(const unsigned long long *__restrict__ incl, int64_t n, int32_t world,
                            int64_t *__restrict__ cuts) {
    const int r = threadIdx.x + 1;  // cuts[1..world-1]
    if (r >= world) return;
    const unsigned long long total = incl[n - 1];
    const unsigned long long want = (unsigned long long)((double)total * r / world);
    int64_t lo = 0, hi = n;  // first v with incl[v] > want ... vertices [0, v] hold <= want + deg
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (incl[mid] <= want) lo = mid + 1;
        else hi = mid;
    }
    cuts[r] = lo;
}

void slpa_rmat_cuts_impl(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB, uint32_t tABC,
                         uint64_t seed, int32_t permute, uint64_t perm_key, int32_t world, int64_t *cuts_out) {
    SLPA_REQUIRE(scale >= 1 && scale <= 31, SLPA_EINVAL, "rmat scale must be in [1, 31]");
    SLPA_REQUIRE(world >= 1 && world <= 1024, SLPA_EINVAL, "world must be in [1, 1024]");
    const int64_t n = 1LL << scale;
    cudaStream_t s = ctx->stream;
    const int64_t chunk = std::min<int64_t>(std::max<int64_t>(num_edges, 1), 1LL << 27);
    DevBuf<uint64_t> buf;
    DevBuf<unsigned long long> deg, incl;
    DevBuf<int64_t> cuts;
    buf.alloc(chunk);
    deg.alloc(n);
    incl.alloc(n);
    cuts.alloc(world + 1);
    CUDA_TRY(cudaMemsetAsync(deg.p, 0, (size_t)n * sizeof(unsigned long long), s));
    for (int64_t e0 = 0; e0 < num_edges; e0 += chunk) {
        const int64_t cnt = std::min(chunk, num_edges - e0);
        k_gen_rmat<<<grid_for(cnt, kT), kT, 0, s>>>(scale, e0, cnt, tA, tAB, tABC, seed, permute, perm_key,
                                                    drop_key(n), buf.p);
        k_key_degrees<<<grid_for(cnt, kT), kT, 0, s>>>(buf.p, cnt, drop_key(n), deg.p);
        CUDA_TRY(cudaGetLastError());
    }
    unsigned long long *in = deg.p, *out = incl.p;
    const int64_t nn = n;
    cub_call(ctx, [&](void *tmp, size_t &bytes) { return cub::DeviceScan::InclusiveSum(tmp, bytes, in, out, nn, s); });
    std::vector<int64_t> h((size_t)world + 1, 0);
    h[world] = n;
    CUDA_TRY(cudaMemcpyAsync(cuts.p, h.data(), h.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (world > 1) k_find_cuts<<<1, 1024, 0, s>>>(incl.p, n, world, cuts.p);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(h.data(), cuts.p, h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int r = 1; r <= world; ++r) h[r] = std::max(h[r], h[r - 1]);  // monotone
    std::copy(h.begin(), h.end(), cuts_out);
}

// One rank's rows of the RMAT graph: every rank generates the
// same edge stream (counter-based RNG) in chunks, keeps the pairs touching
// its vertex range, and assembles only arcs whose source it owns.  Offsets
// stay global (n+1, rows outside the range empty), targets are global ids.
void slpa_part_gen_rmat_impl(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB,
                             uint32_t tABC, uint64_t seed, int32_t permute, uint64_t perm_key, int64_t r0,
                             int64_t r1) {
    SLPA_REQUIRE(scale >= 1 && scale <= 31, SLPA_EINVAL, "rmat scale must be in [1, 31]");
    const int64_t n = 1LL << scale;
    SLPA_REQUIRE(r0 >= 0 && r0 <= r1 && r1 <= n, SLPA_EINVAL, "bad vertex range");
    cudaStream_t s = ctx->stream;
    const int64_t chunk = std::min<int64_t>(num_edges, 1LL << 27);
    DevBuf<uint64_t> buf, kept, sel;
    DevBuf<int64_t> nsel;
    buf.alloc(chunk);
    nsel.alloc(1);
    std::vector<DevBuf<uint64_t>> parts;
    int64_t total = 0;
    std::vector<int64_t> sizes;
    for (int64_t e0 = 0; e0 < num_edges; e0 += chunk) {
        const int64_t cnt = std::min(chunk, num_edges - e0);
        k_gen_rmat<<<grid_for(cnt, kT), kT, 0, s>>>(scale, e0, cnt, tA, tAB, tABC, seed, permute, perm_key,
                                                    drop_key(n), buf.p);
        CUDA_TRY(cudaGetLastError());
        DevBuf<uint64_t> out;
        out.alloc(cnt);
        uint64_t *in = buf.p, *o = out.p;
        int64_t *ns = nsel.p;
        TouchesRange pred{r0, r1};
        cub_call(ctx, [&](void *tmp, size_t &bytes) { return cub::DeviceSelect::If(tmp, bytes, in, o, ns, cnt, pred, s); });
        int64_t h = 0;
        CUDA_TRY(cudaMemcpyAsync(&h, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        parts.push_back(DevBuf<uint64_t>());
        parts.back().p = out.p;
        parts.back().count = out.count;
        out.p = nullptr;
        out.count = 0;
        sizes.push_back(h);
        total += h;
    }
    buf.release();
    kept.alloc(total + 1);
    int64_t off = 0;
    for (size_t i = 0; i < parts.size(); ++i) {
        if (sizes[i]) CUDA_TRY(cudaMemcpyAsync(kept.p + off, parts[i].p, sizes[i] * sizeof(uint64_t),
                                               cudaMemcpyDeviceToDevice, s));
        off += sizes[i];
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    for (auto &p : parts) p.release();
    assemble_from_keys(ctx, n, kept, total, key_end_bit(n), r0, r1);
}
