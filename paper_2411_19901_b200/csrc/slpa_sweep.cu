// slpa_sweep.cu -- one label-propagation sweep on the B200.
//
// Reference semantics (lpa.py:204-224): vertices are visited in order; an
// unprocessed vertex clears its flag, selects a candidate from its
// neighbours' CURRENT labels (earlier vertices' updates of this sweep are
// visible), adopts it when it differs (and, in pick-less sweeps, is
// smaller), and then marks all its out-neighbours unprocessed.
//
// Deterministic mode (worker_count == 0) reproduces that sequential sweep
// bit-exactly with speculative rounds:
//   * vertex v's inputs are L1[u] of lower-positioned neighbours u (the
//     labels they end the sweep with) and L0[u] of higher ones;
//   * v takes its turn iff F0[v] or some lower in-neighbour changed;
//   * the map (inputs -> output) is acyclic in position, so its fixpoint is
//     unique and equals the sequential sweep.  Round 0 evaluates every
//     flagged vertex against the current estimates; any vertex whose output
//     (label, changed bit) moves re-queues its higher-positioned dependants
//     (dirty bitmap); rounds repeat until no output moves.
//   * L1 and the changed bit share one 32-bit word (bit 31), so a single
//     gather of a lower neighbour gives its label and whether it changed.
// Async mode (worker_count > 0) is the paper's in-place parallel sweep.
#include <algorithm>
#include <climits>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>
#include <cstdlib>
#include "slpa_eval.cuh"

namespace {

// Next-round worklists from one pass over the dirty bitmap (1, default) or
// from passes over every degree bin (0); rounds with more light vertices
// than scan_sort_min() re-derive the degree-ordered list from the bins.
int scan_mode() {
    static const int m = [] {
        const char *e = getenv("SLPA_SCAN");
        return e ? atoi(e) : 1;
    }();
    return m;
}
int64_t scan_sort_min() {
    static const int64_t m = [] {
        const char *e = getenv("SLPA_SCAN_SORT_MIN");
        return e ? atoll(e) : 32768LL;
    }();
    return m;
}

// High-degree rounds with at most this many vertices use the block-per-vertex
// slot-parallel scan (short chains) instead of the warp-per-vertex one.
int64_t hi_small_max() {
    static const int64_t m = [] {
        const char *e = getenv("SLPA_HI_SMALL");
        return e ? atoll(e) : 16384LL;
    }();
    return m;
}

// Low-degree rounds with at most this many vertices use the warp-per-vertex
// kernel.
int64_t lo_small_max() {
    static const int64_t m = [] {
        const char *e = getenv("SLPA_LO_SMALL");
        return e ? atoll(e) : 2048LL;
    }();
    return m;
}

// Light-vertex commit in position order (1, default) or over the bin (0).
int commit_pos_mode() {
    static const int m = [] {
        const char *e = getenv("SLPA_COMMIT_POS");
        return e ? atoi(e) : 1;
    }();
    return m;
}

// Round 0 of a deterministic sweep launches the light vertices from a
// flag-compacted copy of their bin (1, default) or over the whole bin (0).
int round0_compact() {
    static const int m = [] {
        const char *e = getenv("SLPA_R0_COMPACT");
        return e ? atoi(e) : 1;
    }();
    return m;
}

// Giants run asynchronously across rounds (1, default) or are joined every
// round (0).
int giant_async_mode() {
    static const int m = [] {
        const char *e = getenv("SLPA_GIANT_ASYNC");
        return e ? atoi(e) : 1;
    }();
    return m;
}

// Heavy (deferred) vertices run once the light worklist is at most this size
// (default: 1/256 of the light vertices, >= 1024; measured at RMAT s24 the
// light tail rounds then overlap the heavy round instead of preceding it).
int64_t defer_min(int64_t n_light) {
    static const int64_t m = [] {
        const char *e = getenv("SLPA_DEFER_MIN");
        return e ? atoll(e) : -1LL;
    }();
    return m >= 0 ? m : std::max<int64_t>(1024, n_light / 256);
}

// SLPA_TRACE=1: per-round worklist sizes on stderr (diagnostics only).
struct TimelineEv {
    int cls;
    bool giant;
    cudaEvent_t e0, e1;
};
std::vector<TimelineEv> &timeline() {
    static std::vector<TimelineEv> t;
    return t;
}

int trace_rounds() {
    static const int t = [] {
        const char *e = getenv("SLPA_TRACE");
        return e ? atoi(e) : 0;
    }();
    return t;
}

// ================================================================== round plumbing
// Round 0 with heavy vertices deferred from the start: flagged heavy
// vertices go straight to the pending bitmap.
__global__ void __launch_bounds__(kThreads) k_defer_flagged(const int32_t *__restrict__ bin, int64_t count,
                                                            const uint8_t *__restrict__ flags,
                                                            uint32_t *__restrict__ pend) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int32_t v = __ldg(&bin[i]);
    if (flags[v]) atomicOr(&pend[v >> 5], 1u << (v & 31));
}

// Deferred heavy (mid / hi) vertices: their dirty bits move to a persistent
// pending bitmap and are only re-evaluated once the light vertices are quiet.
__global__ void __launch_bounds__(kThreads) k_defer_dirty(const int32_t *__restrict__ bin, int64_t count,
                                                          const uint32_t *__restrict__ dirty,
                                                          uint32_t *__restrict__ pend) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int32_t v = __ldg(&bin[i]);
    if ((__ldcg(&dirty[v >> 5]) >> (v & 31)) & 1u) atomicOr(&pend[v >> 5], 1u << (v & 31));
}

// Next-round worklist = the entries of a degree-ordered bin whose dirty bit
// is set (so re-evaluation warps stay degree-homogeneous and the longest
// high-degree scans start first).  One atomic per block; order within a
// block is kept.  The bitmap is cleared afterwards by a memset.
__global__ void __launch_bounds__(kThreads) k_filter_dirty(const int32_t *__restrict__ bin, int64_t count,
                                                           const uint32_t *__restrict__ dirty,
                                                           int32_t *__restrict__ out,
                                                           unsigned long long *__restrict__ cursor, int as_index) {
    __shared__ int s_warp[kThreads / 32];
    __shared__ unsigned long long s_base;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t v = 0;
    bool hit = false;
    if (i < count) {
        v = __ldg(&bin[i]);
        hit = (__ldcg(&dirty[v >> 5]) >> (v & 31)) & 1u;
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) s_warp[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int j = 0; j < kThreads / 32; ++j) {
            int c = s_warp[j];
            s_warp[j] = tot;
            tot += c;
        }
        s_base = tot ? atomicAdd(cursor, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    if (hit) out[s_base + s_warp[w] + __popc(m & ((1u << lane) - 1))] = as_index ? (int32_t)i : v;
}

// Next-sweep flag marks go to a bitmap (n/32 words, L2-resident) with one
// atomicOr each instead of random byte stores into the n-byte flag array;
// k_flag_bits_to_bytes then writes the byte flags in one coalesced pass.
__device__ __forceinline__ void mark_flag(const SweepArgs &a, int32_t t) {
    atomicOr(&a.fbits[t >> 5], 1u << (t & 31));
}

__global__ void k_flag_bits_to_bytes(const uint32_t *__restrict__ bits, uint8_t *__restrict__ bytes, int64_t n) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;  // 4 flags per thread
    if (i >= n) return;
    const uint32_t w = (__ldg(&bits[i >> 5]) >> (i & 31)) & 0xfu;
    if (i + 4 <= n) {
        const uint32_t x = (w & 1u) | ((w & 2u) << 7) | ((w & 4u) << 14) | ((w & 8u) << 21);
        *reinterpret_cast<uint32_t *>(bytes + i) = x;
    } else {
        for (int64_t j = i; j < n; ++j) bytes[j] = (uint8_t)((w >> (j - i)) & 1u);
    }
}

// End of a deterministic sweep: fold L1 into L0, count ΔN, and set the
// next sweep's flags: a changed u marks its out-neighbours t with
// pos(t) <= pos(u) (those whose turn has passed; lpa.py:223).
__global__ void __launch_bounds__(kThreads) k_commit_lo(SweepArgs a, const int32_t *__restrict__ list, int64_t count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long d = 0;
    if (i < count) {
        const int32_t v = __ldg(&list[i]);
        uint32_t wv = a.lab_new[v];
        if (wv & SLPA_CHG) {
            int32_t c = (int32_t)(wv & SLPA_LMASK);
            a.lab_old[v] = c;
            a.lab_new[v] = (uint32_t)c;
            d = 1;
            const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
            for (int64_t e0 = lo; e0 < hi; e0 += 8) {  // 8 independent target loads in flight
                int32_t t[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) t[j] = e0 + j < hi ? __ldg(&a.tgt[e0 + j]) : INT32_MAX;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (t[j] <= v) mark_flag(a, t[j]);
            }
        }
    }
    warp_count(a.counters, 0, 0, d);
}

__global__ void __launch_bounds__(kThreads) k_commit_hi(SweepArgs a, const int32_t *__restrict__ list, int64_t count,
                                                     bool marks = true) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= count) return;
    const int32_t v = __ldg(&list[wid]);
    uint32_t wv = a.lab_new[v];
    if (!(wv & SLPA_CHG)) return;
    if (marks) {
        const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
#pragma unroll 4
        for (int64_t e = lo + lane; e < hi; e += 32) {
            int32_t t = __ldg(&a.tgt[e]);
            if (t <= v) mark_flag(a, t);
        }
    }
    __syncwarp();
    if (lane == 0) {
        int32_t c = (int32_t)(wv & SLPA_LMASK);
        a.lab_old[v] = c;
        a.lab_new[v] = (uint32_t)c;
        ctr_add(a.counters, CNT_DELTA, 1ull);
    }
}

// The giants' next-sweep marks: one warp walking a row of ~4e5 arcs is a
// chain of dependent load rounds (measured 3.4 ms for sweep 1's commit at
// RMAT s24), so the rows are cut into kCommitArcs slices, a block each
// (blockIdx.y = giant).  k_commit_hi(marks = false) then commits the labels.
constexpr int kCommitArcs = 4096;
__global__ void __launch_bounds__(kThreads) k_commit_marks_wide(SweepArgs a, const int32_t *__restrict__ list) {
    const int32_t v = __ldg(&list[blockIdx.y]);
    if (!(__ldcg(&a.lab_new[v]) & SLPA_CHG)) return;
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int64_t b = lo + (int64_t)blockIdx.x * kCommitArcs;
    if (b >= hi) return;
    const int64_t end = b + kCommitArcs < hi ? b + kCommitArcs : hi;
#pragma unroll 4
    for (int64_t e = b + threadIdx.x; e < end; e += kThreads) {
        const int32_t t = __ldg(&a.tgt[e]);
        if (t <= v) mark_flag(a, t);
    }
}

__global__ void k_init_labels(int32_t *lab_old, uint32_t *lab_new, uint8_t *flags, const int32_t *ids, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t l = ids ? ids[i] : (int32_t)i;
    lab_old[i] = l;
    if (lab_new) lab_new[i] = (uint32_t)l;
    flags[i] = 1;
}

__global__ void k_clear_isolated_flags(uint8_t *flags, const uint8_t *cls, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && cls[i] == CLS_NONE) flags[i] = 0;
}

// by-position <-> by-id permutations for host I/O
__global__ void k_pos_to_id_i32(const int32_t *src, int32_t *dst, const int32_t *ids, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[ids[i]] = src[i];
}
__global__ void k_id_to_pos_i32(const int32_t *src, int32_t *dst, const int32_t *ids, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[ids[i]];
}
__global__ void k_pos_to_id_u8(const uint8_t *src, uint8_t *dst, const int32_t *ids, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[ids[i]] = src[i];
}
__global__ void k_id_to_pos_u8(const uint8_t *src, uint8_t *dst, const int32_t *ids, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[ids[i]] ? 1 : 0;
}
__global__ void k_norm_flags(uint8_t *f, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) f[i] = f[i] ? 1 : 0;
}
__global__ void k_sync_lab_new(const int32_t *lab_old, uint32_t *lab_new, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) lab_new[i] = (uint32_t)lab_old[i];
}

// ------------------------------------------------------------------ dispatch
// Integer sketch values when the exactness precondition holds (slpa_sketch.cuh).
KernelSet kernels_for(const slpa_ctx *ctx, const slpa_config *cfg, bool det) {
    static const int force_fp64 = [] {
        const char *e = getenv("SLPA_FORCE_FP64");
        return e ? atoi(e) : 0;
    }();
    const bool iv = ctx->g.int_weights && !force_fp64;
    if (ctx->g.w_f64) {
        if (iv) return det ? slpa_pick_f64_u32_det(cfg) : slpa_pick_f64_u32_async(cfg);
        return det ? slpa_pick_f64_f64_det(cfg) : slpa_pick_f64_f64_async(cfg);
    }
    if (iv) return det ? slpa_pick_f32_u32_det(cfg) : slpa_pick_f32_u32_async(cfg);
    return det ? slpa_pick_f32_f64_det(cfg) : slpa_pick_f32_f64_async(cfg);
}

SweepArgs make_args(slpa_ctx *ctx, const slpa_config *cfg, int pickless) {
    ctx->cur_cfg = cfg;
    ctx->wb.wl_mid.alloc(ctx->g.n_mid + 1);  // worklists sized by the current bins (no-op when large enough)
    ctx->wb.wl_hi.alloc(ctx->g.n_hi + 1);
    SweepArgs a{};
    DeviceGraph &g = ctx->g;
    a.off = g.off();
    a.tgt = g.tgt();
    a.w = g.w();
    a.roff = g.symmetric ? nullptr : g.roff.p;
    a.rsrc = g.symmetric ? nullptr : g.rsrc.p;
    a.cls = g.cls.p;
    a.lab_old = ctx->wb.lab_old.p;
    a.lab_new = ctx->wb.lab_new.p;
    a.flag_cur = ctx->wb.flag_a.p;
    a.flag_next = ctx->wb.flag_b.p;
    a.dirty_next = ctx->wb.dirty_a.p;
    a.counters = ctx->wb.counters.p;
    a.pickless = pickless;
    a.k = cfg->sketch_slots;
    a.parts = cfg->partial_groups;
    a.scan_double = cfg->scan_mode == SLPA_SCAN_DOUBLE;
    a.symmetric = g.symmetric;
    a.thr = cfg->degree_threshold;
    a.single = cfg->variant == SLPA_VARIANT_MG && cfg->shared_sketch;
    a.tbits = ctx->prof_on ? ctx->wb.tbits.p : nullptr;
    a.fbits = ctx->wb.fbits.p;
    a.zkey = ctx->zkey;
    a.giant_bin = g.bin_giant.p;
    a.giant_off = g.giant_off.p;
    a.glab = ctx->wb.glab.p;
    a.gw = ctx->wb.gw.p;
    return a;
}

void read_counters(slpa_ctx *ctx) {
    CUDA_TRY(cudaMemcpyAsync(ctx->h_counters, ctx->wb.counters.p, CNT_TOTAL * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    for (int c = 0; c < CNT_N; ++c) {
        unsigned long long s = 0;
        for (int j = 0; j < CNT_STRIPES; ++j) s += ctx->h_counters[c * CNT_STRIPES + j];
        ctx->h_sum[c] = s;
    }
}

// Profiling mode (slpa_set_profiling): CUDA events on the context stream
// around every launch, attributed to a kernel class with the vertices and
// arcs that launch evaluated.  Off by default (no host syncs added).
template <class F>
void timed_launch(slpa_ctx *ctx, int cls, int nlaunch, F &&fn, cudaStream_t st = nullptr) {
    ctx->stats.kernel_launches += nlaunch;
    if (!ctx->prof_on) {
        if (trace_rounds() >= 3) {  // timeline: events around the launch, read at the end of the sweep
            cudaStream_t es = st ? st : ctx->stream;
            TimelineEv ev;
            ev.cls = cls;
            CUDA_TRY(cudaEventCreate(&ev.e0));
            CUDA_TRY(cudaEventCreate(&ev.e1));
            CUDA_TRY(cudaEventRecord(ev.e0, es));
            fn();
            CUDA_TRY(cudaEventRecord(ev.e1, es));
            ev.giant = st != nullptr && st != ctx->stream;
            timeline().push_back(ev);
            return;
        }
        fn();
        return;
    }
    unsigned long long e0 = ctx->h_sum[CNT_EVALS] + ctx->h_sum[CNT_EVALS_HI];
    unsigned long long a0 = ctx->h_sum[CNT_ARCS] + ctx->h_sum[CNT_ARCS_HI];
    CUDA_TRY(cudaEventRecord(ctx->pev0, ctx->stream));
    fn();
    CUDA_TRY(cudaEventRecord(ctx->pev1, ctx->stream));
    CUDA_TRY(cudaEventSynchronize(ctx->pev1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, ctx->pev0, ctx->pev1));
    read_counters(ctx);
    ctx->prof.launches[cls] += nlaunch;
    ctx->prof.ms[cls] += ms;
    ctx->prof.evals[cls] += (int64_t)(ctx->h_sum[CNT_EVALS] + ctx->h_sum[CNT_EVALS_HI] - e0);
    ctx->prof.arcs[cls] += (int64_t)(ctx->h_sum[CNT_ARCS] + ctx->h_sum[CNT_ARCS_HI] - a0);
    if (trace_rounds() >= 2)
        fprintf(stderr, "[slpa]   launch class %d: %.3f ms, %lld evals, %lld arcs\n", cls, ms,
                (long long)(ctx->h_sum[CNT_EVALS] + ctx->h_sum[CNT_EVALS_HI] - e0),
                (long long)(ctx->h_sum[CNT_ARCS] + ctx->h_sum[CNT_ARCS_HI] - a0));
}

// Largest degree of the resident graph (exact / large-k scratch sizing).
__global__ void k_max_degree(const int64_t *__restrict__ off, int64_t n, unsigned long long *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long d = i < n ? (unsigned long long)(__ldg(&off[i + 1]) - __ldg(&off[i])) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, d, o);
        d = x > d ? x : d;
    }
    if ((threadIdx.x & 31) == 0 && d) atomicMax(out, d);
}

int64_t graph_max_degree(slpa_ctx *ctx) {
    DeviceGraph &g = ctx->g;
    if (g.max_deg >= 0) return g.max_deg;
    WorkBuffers &wb = ctx->wb;
    wb.dcount.alloc(2);
    CUDA_TRY(cudaMemsetAsync(wb.dcount.p, 0, sizeof(unsigned long long), ctx->stream));
    if (g.n > 0) k_max_degree<<<grid_for(g.n, kThreads), kThreads, 0, ctx->stream>>>(g.off(), g.n, wb.dcount.p);
    CUDA_TRY(cudaGetLastError());
    unsigned long long h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, wb.dcount.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    g.max_deg = (int64_t)h;
    return g.max_deg;
}

// Scratch of the exact (xmode 1) and large-k (xmode 2) kernels.
//  exact: open-addressing tables (int32 keys, binary64 totals) of 2^26 slots
//    in all, kept empty (key -1, total 0.0; the kernel clears the slots it
//    used).  Two launches: vertices of degree <= 4096 with 8192-slot regions
//    per warp (thousands of warps), larger ones with regions sized for the
//    largest degree (a few warps);
//  large k: two k-slot sketches per thread, a fixed number of threads (at
//    most ~1 GiB) striding over the worklist.
constexpr int64_t kExactSmallDeg = 4096;

void setup_xscratch_bigk(slpa_ctx *ctx, const slpa_config *cfg, SweepArgs &a) {
    const size_t budget = (size_t)1 << 30;
    const size_t vb = ctx->g.int_weights ? 4 : 8;
    const size_t per_unit = (size_t)cfg->sketch_slots * 2 * (4 + vb);
    int64_t units = std::min<int64_t>((int64_t)ctx->num_sms * 64, (int64_t)(budget / per_unit));
    units = std::max<int64_t>(32, units / 32 * 32);
    const size_t need = per_unit * (size_t)units;
    if (ctx->wb.xscratch.count < need) ctx->wb.xscratch.alloc(need);
    ctx->xs_key = 0;  // the exact tables' contents are gone
    a.xs = ctx->wb.xscratch.p;
    a.xunits = units;
}

void setup_xscratch_exact(slpa_ctx *ctx) {
    int64_t cap_big = 64;
    while (cap_big < 2 * std::max<int64_t>(graph_max_degree(ctx), 1)) cap_big <<= 1;
    const int64_t slots = std::max<int64_t>((int64_t)1 << 26, cap_big);
    if (ctx->xs_key != slots) {
        ctx->wb.xscratch.alloc((size_t)slots * 4);
        ctx->wb.xtotals.alloc((size_t)slots);
        CUDA_TRY(cudaMemsetAsync(ctx->wb.xscratch.p, 0xff, (size_t)slots * 4, ctx->stream));
        CUDA_TRY(cudaMemsetAsync(ctx->wb.xtotals.p, 0, (size_t)slots * 8, ctx->stream));
        ctx->xs_key = slots;
    }
}

void launch_lane(slpa_ctx *ctx, const KernelSet &ks, int which, const SweepArgs &a0, const int32_t *list, int64_t cnt,
                 int round0, int cls, bool allow_small = false) {
    if (cnt <= 0) return;
    const EvalKernel k = which == 0 ? ks.lo : ks.mid;
    const int threads = ks.lo_threads;
    if (ks.xmode == 2) {
        SweepArgs a = a0;
        setup_xscratch_bigk(ctx, ctx->cur_cfg, a);
        timed_launch(ctx, cls, 1, [&] {
            k<<<grid_for(a.xunits, threads), threads, 0, ctx->stream>>>(a, list, cnt, round0);
            CUDA_TRY(cudaGetLastError());
        });
        return;
    }
    if (ks.xmode == 1) {
        setup_xscratch_exact(ctx);
        const int64_t slots = ctx->xs_key, maxdeg = graph_max_degree(ctx);
        for (int tier = 0; tier < 2; ++tier) {
            SweepArgs a = a0;
            int64_t cap = 64;
            if (tier == 0) {
                cap = 2 * kExactSmallDeg;
                a.xdeg_lo = -1;
                a.xdeg_hi = kExactSmallDeg;
            } else {
                if (maxdeg <= kExactSmallDeg) break;
                while (cap < 2 * maxdeg) cap <<= 1;
                a.xdeg_lo = kExactSmallDeg;
                a.xdeg_hi = INT64_MAX;
            }
            a.xs = ctx->wb.xscratch.p;
            a.xtot = ctx->wb.xtotals.p;
            a.xcap = cap;
            a.xunits = std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * 64, slots / cap));
            timed_launch(ctx, cls, 1, [&] {
                k<<<grid_for(a.xunits * 32, threads), threads, 0, ctx->stream>>>(a, list, cnt, round0);
                CUDA_TRY(cudaGetLastError());
            });
        }
        return;
    }
    const EvalKernel small = (allow_small && which == 0) ? ks.lo_small : nullptr;
    if (small && cnt <= lo_small_max()) {  // few vertices: a warp per vertex (latency, not volume)
        timed_launch(ctx, cls, 1, [&] {
            small<<<grid_for(cnt * 32, kThreads), kThreads, 0, ctx->stream>>>(a0, list, cnt, round0);
            CUDA_TRY(cudaGetLastError());
        });
        return;
    }
    timed_launch(ctx, cls, 1, [&] {
        k<<<grid_for(cnt, threads), threads, 0, ctx->stream>>>(a0, list, cnt, round0);
        CUDA_TRY(cudaGetLastError());
    });
}

// High-degree rounds.  The scan / merge / finish split stages 2 KB of part
// sketches per vertex; large rounds run in slices of kHiSlice vertices so the
// scratch stays at kHiSlice x 2 KB (128 MB) instead of scaling with the bin
// (1.1 GB at RMAT s24).  Any evaluation order within a round reaches the same
// fixpoint; a later slice simply sees an earlier one's labels.
// Heavy rounds run in slices of this many vertices (part-sketch scratch =
// slice x 2 KB).  Measured at RMAT s24: 64k 58.4 ms, 128k 56.0, 256k 54.4,
// 512k 54.1 ms per run (fewer scan -> merge -> finish tails); 256k costs a
// fixed 512 MB of scratch.
int64_t hi_slice() {
    static const int64_t m = [] {
        const char *e = getenv("SLPA_HI_SLICE");
        return e ? std::max<int64_t>(1, atoll(e)) : 262144LL;
    }();
    return m;
}

// Commit of the giant bin: wide marks, then the labels.
void commit_giants(slpa_ctx *ctx, const SweepArgs &a, cudaStream_t s) {
    const DeviceGraph &g = ctx->g;
    const int64_t slices = std::max<int64_t>(1, (g.giant_max_deg + kCommitArcs - 1) / kCommitArcs);
    k_commit_marks_wide<<<dim3((unsigned)slices, (unsigned)g.n_giant), kThreads, 0, s>>>(a, g.bin_giant.p);
    k_commit_hi<<<grid_for(g.n_giant * 32, kThreads), kThreads, 0, s>>>(a, g.bin_giant.p, g.n_giant, false);
}

void launch_hi(slpa_ctx *ctx, const KernelSet &ks, const SweepArgs &a, const int32_t *list, int64_t cnt, int round0,
               int cls) {
    if (cnt <= 0) return;
    SweepArgs aa = a;
    const bool small = ks.hi_small && cnt <= hi_small_max();
    if (ks.hi_merge && !small) {
        WorkBuffers &wb = ctx->wb;
        const int64_t kHiSlice = hi_slice();
        const int64_t cap = std::min<int64_t>(std::max<int64_t>(ctx->g.n_hi, 1), kHiSlice);
        wb.hparts.alloc((size_t)cap * kLpmWords);
        wb.hmeta.alloc((size_t)cap);
        aa.hparts = wb.hparts.p;
        aa.hmeta = wb.hmeta.p;
    }
    if (small) {  // fused block-per-vertex kernel (merge + finish inside)
        timed_launch(ctx, cls, 1, [&] {
            ks.hi_small<<<(unsigned)cnt, kGiantWarps * 32, 0, ctx->stream>>>(aa, list, cnt, round0);
            CUDA_TRY(cudaGetLastError());
        });
        return;
    }
    if (!ks.hi_merge) {
        timed_launch(ctx, cls, 1, [&] {
            const int64_t items = ks.hi_vpw ? (cnt + ks.hi_vpw - 1) / ks.hi_vpw * 32 : cnt;
            ks.hi<<<grid_for(items, ks.hi_threads), ks.hi_threads, 0, ctx->stream>>>(aa, list, cnt, round0);
            CUDA_TRY(cudaGetLastError());
        });
        return;
    }
    const int64_t kHiSlice = hi_slice();
    for (int64_t b = 0; b < cnt; b += kHiSlice) {
        const int64_t c = std::min(kHiSlice, cnt - b);
        const int32_t *l = list + b;
        timed_launch(ctx, cls, 3, [&] {
            ks.hi<<<grid_for(c * 32, ks.hi_threads), ks.hi_threads, 0, ctx->stream>>>(aa, l, c, round0);
            ks.hi_merge<<<grid_for(c, kThreads), kThreads, 0, ctx->stream>>>(aa, l, c, round0);
            ks.hi_finish<<<grid_for(c * 32, kThreads), kThreads, 0, ctx->stream>>>(aa, l, c, round0);
            CUDA_TRY(cudaGetLastError());
        });
    }
}

// Giants: gather then replay; `slots` index bin_giant.  They are a handful
// of warps, so (outside profiling) they run on a second stream, overlapping
// the other kernels of the round; giant_join() makes the main stream wait.
void launch_giant(slpa_ctx *ctx, const KernelSet &ks, const SweepArgs &a, const int32_t *slots, int64_t cnt,
                  int round0) {
    if (cnt <= 0 || !ks.gather) return;
    const bool overlap = !ctx->prof_on;
    cudaStream_t gs = overlap ? ctx->stream2 : ctx->stream;
    if (overlap) {
        CUDA_TRY(cudaEventRecord(ctx->gev0, ctx->stream));
        CUDA_TRY(cudaStreamWaitEvent(gs, ctx->gev0, 0));
    }
    timed_launch(ctx, SLPA_PROF_EVAL_GIANT, 2, [&] {
        const dim3 grid((unsigned)((ctx->g.giant_max_deg + kGatherArcs - 1) / kGatherArcs), (unsigned)cnt);
        ks.gather<<<grid, kGatherThreads, 0, gs>>>(a, slots, cnt, round0);
        if (ks.giant_threads)
            ks.giant<<<(unsigned)cnt, ks.giant_threads, 0, gs>>>(a, slots, cnt, round0);
        else
            ks.giant<<<grid_for(cnt * 32, kWinThreads), kWinThreads, 0, gs>>>(a, slots, cnt, round0);
        CUDA_TRY(cudaGetLastError());
    }, gs);
    if (overlap) {
        CUDA_TRY(cudaEventRecord(ctx->gev1, gs));
        ctx->giant_pending = 1;
    }
}

void giant_join(slpa_ctx *ctx) {
    if (ctx->giant_pending) {
        CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->gev1, 0));
        ctx->giant_pending = 0;
    }
}

void launch_filter(cudaStream_t s, const int32_t *bin, int64_t count, const uint32_t *dirty, int32_t *out,
                   unsigned long long *cursor, int as_index = 0) {
    if (count <= 0) return;
    k_filter_dirty<<<grid_for(count, kThreads), kThreads, 0, s>>>(bin, count, dirty, out, cursor, as_index);
}

// One pass over the dirty bitmap instead of a pass over every degree bin:
// thread i takes word i, reads the 32 degree classes of its vertices with one
// 256-bit load, appends the light ones to the next low-degree worklist
// (ascending position; one atomic per warp) and moves the heavy ones to the
// pending bitmap (the deferral of k_defer_dirty).  The caller may still
// re-derive a degree-ordered low worklist from the bins for large rounds.
__global__ void __launch_bounds__(kThreads) k_scan_dirty(const uint32_t *__restrict__ dirty,
                                                         uint32_t *__restrict__ pend,
                                                         const uint8_t *__restrict__ cls, int64_t nwords,
                                                         int32_t *__restrict__ out,
                                                         unsigned long long *__restrict__ cursor,
                                                         uint32_t *__restrict__ pend_g,
                                                         unsigned long long *__restrict__ new_g) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    uint32_t w = i < nwords ? __ldcg(&dirty[i]) : 0u;
    uint32_t lom = 0, hvm = 0, gm = 0;
    if (w) {
        uint32_t c[8];
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7])
                     : "l"(cls + i * 32));
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            const uint32_t cb = (c[b >> 2] >> ((b & 3) * 8)) & 0xffu;
            const uint32_t bit = 1u << b;
            if (w & bit) {
                if (cb == CLS_LO) lom |= bit;
                else if (cb == CLS_GIANT && pend_g) gm |= bit;
                else hvm |= bit;
            }
        }
        if (hvm) atomicOr(&pend[i], hvm);
        if (gm) {  // asynchronous giants: their own pending set, counted when new
            const uint32_t old = atomicOr(&pend_g[i], gm);
            if (gm & ~old) atomicAdd(new_g, (unsigned long long)__popc(gm & ~old));
        }
    }
    const int cnt = __popc(lom);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(cursor, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    int pos = (int)base + incl - cnt;
    while (lom) {
        const int b = __ffs(lom) - 1;
        lom &= lom - 1;
        out[pos++] = (int32_t)(i * 32 + b);
    }
}

// Asynchronous giants: OR a finished batch's dependant marks into the round
// bitmap and clear them; move a class's round-0 deferral bits to its own set.
__global__ void k_or_clear(uint32_t *__restrict__ src, uint32_t *__restrict__ dst, int64_t nwords) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nwords) return;
    const uint32_t w = src[i];
    if (w) {
        atomicOr(&dst[i], w);
        src[i] = 0;
    }
}
__global__ void k_move_class(const int32_t *__restrict__ bin, int64_t count, uint32_t *__restrict__ from,
                             uint32_t *__restrict__ to) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int32_t v = __ldg(&bin[i]);
    const uint32_t bit = 1u << (v & 31);
    if (atomicAnd(&from[v >> 5], ~bit) & bit) atomicOr(&to[v >> 5], bit);
}

// Round-0 worklist of a later sweep: the flagged entries of a degree-ordered
// bin, order kept within a block (one atomic per block).
__global__ void __launch_bounds__(kThreads) k_filter_flags(const int32_t *__restrict__ bin, int64_t count,
                                                           const uint8_t *__restrict__ flags,
                                                           int32_t *__restrict__ out,
                                                           unsigned long long *__restrict__ cursor) {
    __shared__ int s_warp[kThreads / 32];
    __shared__ unsigned long long s_base;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t v = 0;
    bool hit = false;
    if (i < count) {
        v = __ldg(&bin[i]);
        hit = flags[v] != 0;
    }
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) s_warp[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int j = 0; j < kThreads / 32; ++j) {
            const int c = s_warp[j];
            s_warp[j] = tot;
            tot += c;
        }
        s_base = tot ? atomicAdd(cursor, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    if (hit) out[s_base + s_warp[w] + __popc(m & ((1u << lane) - 1))] = v;
}

// Commit of the light vertices in position order (coalesced label words):
// a changed light vertex folds L1 into L0 and marks its neighbours t <= v.
__global__ void __launch_bounds__(kThreads) k_commit_lo_pos(SweepArgs a, int64_t n) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long d = 0;
    if (v < n) {
        const uint32_t wv = a.lab_new[v];
        if ((wv & SLPA_CHG) && a.cls[v] == CLS_LO) {
            const int32_t c = (int32_t)(wv & SLPA_LMASK);
            a.lab_old[v] = c;
            a.lab_new[v] = (uint32_t)c;
            d = 1;
            const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
            for (int64_t e0 = lo; e0 < hi; e0 += 8) {
                int32_t t[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) t[j] = e0 + j < hi ? __ldg(&a.tgt[e0 + j]) : INT32_MAX;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (t[j] <= v) mark_flag(a, t[j]);
            }
        }
    }
    warp_count(a.counters, 0, 0, d);
}

// Multi-GPU deterministic sweep: dirty marks cross ranks as bytes (NCCL has
// no bitwise-OR reduction; a MAX over 0/1 bytes is the OR).
__global__ void k_dirty_bits_to_bytes(const uint32_t *__restrict__ bits, uint8_t *__restrict__ bytes, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) bytes[i] = (uint8_t)((__ldg(&bits[i >> 5]) >> (i & 31)) & 1u);
}
__global__ void k_dirty_bytes_to_bits(const uint8_t *__restrict__ bytes, uint32_t *__restrict__ bits, int64_t n,
                                      unsigned long long *__restrict__ count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool b = i < n && bytes[i] != 0;
    const unsigned m = __ballot_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0 && i < n) {
        bits[i >> 5] = m;
        if (m) atomicAdd(count, (unsigned long long)__popc(m));
    }
}
// Fold L1 into L0 for every vertex of the replica (owned entries were
// already folded by the commit kernels; this makes the remote ones agree).
__global__ void k_fold_all(int32_t *lab_old, uint32_t *lab_new, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t w = lab_new[i];
    if (w & SLPA_CHG) {
        lab_old[i] = (int32_t)(w & SLPA_LMASK);
        lab_new[i] = w & SLPA_LMASK;
    }
}

// Profiling: vertices the sequential sweep processed (turn bitmap) and their arcs.
// Isolated vertices are never evaluated (no bin); the sequential sweep still
// processes them when flagged (lpa.py:212-214).
__global__ void k_count_turns(const uint32_t *__restrict__ tbits, const int64_t *__restrict__ off,
                              const uint8_t *__restrict__ f0, int64_t n, unsigned long long *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nv = 0, na = 0;
    if (i * 32 < n) {
        const uint32_t w = tbits[i];
        for (int b = 0; b < 32 && i * 32 + b < n; ++b) {
            const int64_t v = i * 32 + b;
            const int64_t d = __ldg(&off[v + 1]) - __ldg(&off[v]);
            if ((w >> b) & 1u) {
                ++nv;
                na += (unsigned long long)d;
            } else if (d == 0 && f0[v]) {
                ++nv;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nv += __shfl_xor_sync(0xffffffffu, nv, o);
        na += __shfl_xor_sync(0xffffffffu, na, o);
    }
    if ((threadIdx.x & 31) == 0 && (nv || na)) {
        atomicAdd(&out[0], nv);
        atomicAdd(&out[1], na);
    }
}

__global__ void k_iota(int32_t *out, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)i;
}

}  // namespace

// ------------------------------------------------------------ multi-GPU deterministic rounds
// The host (distributed.py) drives a partitioned deterministic sweep round by
// round: slpa_part_det_round evaluates this rank's owned vertices (round 0:
// every flagged one; later rounds: the dirty ones) and exports its dirty
// bitmap as bytes; the host all-gathers the owned lab_new ranges and
// MAX-reduces the dirty bytes; slpa_part_det_import turns the global marks
// back into the bitmap.  Every round reads remote labels as of the previous
// exchange -- a stale read is re-evaluated through the dirty marks like any
// other speculation, so the fixpoint is still the sequential sweep.  Heavy
// vertices are not deferred (a round-local policy would need a global vote).
void slpa_part_det_round_impl(slpa_ctx *ctx, const slpa_config *cfg, int pickless, int round) {
    NvtxRange nvtx_round("slpa partitioned round");
    DeviceGraph &g = ctx->g;
    WorkBuffers &wb = ctx->wb;
    cudaStream_t s = ctx->stream;
    const int64_t n = g.n;
    const KernelSet ks = kernels_for(ctx, cfg, true);
    const SweepArgs a = make_args(ctx, cfg, pickless);
    const int64_t nwords = (n + 31) / 32;
    if (round == 0) {
        CUDA_TRY(cudaMemsetAsync(wb.counters.p, 0, CNT_TOTAL * sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(wb.flag_b.p, 0, (size_t)n, s));
        CUDA_TRY(cudaMemsetAsync(wb.dirty_a.p, 0, (size_t)nwords * sizeof(uint32_t), s));
        for (int c = 0; c < CNT_N; ++c) ctx->h_sum[c] = 0;
        if (g.n_giant > 0) {
            k_iota<<<grid_for(g.n_giant, kThreads), kThreads, 0, s>>>(wb.wl_giant.p, g.n_giant);
            launch_giant(ctx, ks, a, wb.wl_giant.p, g.n_giant, 1);
        }
        launch_hi(ctx, ks, a, g.bin_hi.p, g.n_hi, 1, SLPA_PROF_EVAL_HI0);
        launch_lane(ctx, ks, 1, a, g.bin_mid.p, g.n_mid, 1, SLPA_PROF_EVAL_MID0);
        launch_lane(ctx, ks, 0, a, g.bin_lo.p, g.n_lo, 1, SLPA_PROF_EVAL_LO0);
    } else {
        unsigned long long *cur_lo = wb.counters.p + CNT_LO * CNT_STRIPES,
                           *cur_mid = wb.counters.p + CNT_MID * CNT_STRIPES,
                           *cur_hi = wb.counters.p + CNT_HI * CNT_STRIPES,
                           *cur_giant = wb.counters.p + CNT_GIANT * CNT_STRIPES;
        CUDA_TRY(cudaMemsetAsync(cur_lo, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(cur_mid, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(cur_hi, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(cur_giant, 0, sizeof(unsigned long long), s));
        launch_filter(s, g.bin_lo.p, g.n_lo, wb.dirty_a.p, wb.wl_lo.p, cur_lo);
        launch_filter(s, g.bin_hi.p, g.n_hi, wb.dirty_a.p, wb.wl_hi.p, cur_hi);
        launch_filter(s, g.bin_mid.p, g.n_mid, wb.dirty_a.p, wb.wl_mid.p, cur_mid);
        launch_filter(s, g.bin_giant.p, g.n_giant, wb.dirty_a.p, wb.wl_giant.p, cur_giant, 1);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemsetAsync(wb.dirty_a.p, 0, (size_t)nwords * sizeof(uint32_t), s));
        read_counters(ctx);
        const int64_t nlo = (int64_t)ctx->h_sum[CNT_LO], nmid = (int64_t)ctx->h_sum[CNT_MID],
                      nhi = (int64_t)ctx->h_sum[CNT_HI], ngiant = (int64_t)ctx->h_sum[CNT_GIANT];
        launch_giant(ctx, ks, a, wb.wl_giant.p, ngiant, 0);
        launch_hi(ctx, ks, a, wb.wl_hi.p, nhi, 0, SLPA_PROF_EVAL_HIK);
        launch_lane(ctx, ks, 0, a, wb.wl_lo.p, nlo, 0, SLPA_PROF_EVAL_LOK, true);
        launch_lane(ctx, ks, 1, a, wb.wl_mid.p, nmid, 0, SLPA_PROF_EVAL_MIDK);
    }
    giant_join(ctx);
    // no host sync: slpa_part_det_collect (sparse exchange) or
    // slpa_part_det_dense (dense exchange) follows on ctx->stream
    ctx->stats.rounds += 1;
}

// ------------------------------------------------------------ sparse round exchange
// Per round a rank only has to publish (a) the owned label words that moved
// since its last exchange and (b) the dirty marks it set on remote vertices.
// slpa_part_det_collect packs both into one int32 list (words as (id, word)
// pairs, then mark ids); the host all-gathers the lists (padded to the
// longest) and slpa_part_det_apply writes the remote words into the replica
// and sets the marks this rank owns.  When the lists would outweigh the dense
// exchange (4n + n bytes) the host picks slpa_part_det_dense for the round --
// the choice is made from the all-gathered counts, so every rank agrees.
__global__ void k_collect_words(const uint32_t *__restrict__ lab_new, uint32_t *__restrict__ lab_sent, int64_t vb,
                                int64_t ve, int32_t *__restrict__ out, unsigned long long *__restrict__ cursor) {
    const int64_t v = vb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    bool moved = false;
    uint32_t w = 0;
    if (v < ve) {
        w = __ldcg(&lab_new[v]);
        moved = w != lab_sent[v];
        if (moved) lab_sent[v] = w;
    }
    const unsigned m = __ballot_sync(0xffffffffu, moved);
    unsigned long long base = 0;
    if (lane == 0 && m) base = atomicAdd(cursor, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (moved) {
        const int64_t k = (int64_t)base + __popc(m & ((1u << lane) - 1u));
        out[2 * k] = (int32_t)v;
        out[2 * k + 1] = (int32_t)w;
    }
}
__device__ __forceinline__ uint32_t owned_bits(int64_t i, int64_t vb, int64_t ve) {  // word i's owned vertices
    uint32_t own = 0;
    for (int b = 0; b < 32; ++b) {
        const int64_t v = i * 32 + b;
        if (v >= vb && v < ve) own |= 1u << b;
    }
    return own;
}
// remote dirty marks (bitmap words outside the owned range)
__global__ void k_collect_marks(const uint32_t *__restrict__ dirty, int64_t nwords, int64_t vb, int64_t ve,
                                int32_t *__restrict__ out, unsigned long long *__restrict__ cursor) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nwords) return;
    const uint32_t w = dirty[i];
    if (!w) return;
    const uint32_t rem = w & ~owned_bits(i, vb, ve);
    if (!rem) return;
    const unsigned long long base = atomicAdd(cursor, (unsigned long long)__popc(rem));
    int k = 0;
    for (uint32_t r = rem; r; r &= r - 1, ++k) out[base + k] = (int32_t)(i * 32 + __ffs(r) - 1);
}
__global__ void k_apply_lists(const int32_t *__restrict__ recv, int64_t stride, const int64_t *__restrict__ counts,
                              int32_t world, int32_t self, int64_t vb, int64_t ve, uint32_t *__restrict__ lab_new,
                              uint32_t *__restrict__ lab_sent_unused, uint32_t *__restrict__ dirty) {
    const int r = blockIdx.y;
    if (r == self || r >= world) return;
    const int64_t nw = counts[2 * r], nm = counts[2 * r + 1];
    const int32_t *l = recv + (int64_t)r * stride;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nw + nm; x += (int64_t)gridDim.x * blockDim.x) {
        if (x < nw) {
            __stcg(&lab_new[l[2 * x]], (uint32_t)l[2 * x + 1]);
        } else {
            const int32_t t = l[2 * nw + (x - nw)];
            if (t >= vb && t < ve) atomicOr(&dirty[t >> 5], 1u << (t & 31));
        }
    }
}
__global__ void k_clear_remote_bits(uint32_t *__restrict__ dirty, int64_t nwords, int64_t vb, int64_t ve) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nwords && dirty[i]) dirty[i] &= owned_bits(i, vb, ve);
}
__global__ void k_count_owned_bits(const uint32_t *__restrict__ bits, int64_t vb, int64_t ve,
                                   unsigned long long *__restrict__ out) {
    const int64_t v = vb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool b = v < ve && ((__ldcg(&bits[v >> 5]) >> (v & 31)) & 1u);
    const unsigned m = __ballot_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, (unsigned long long)__popc(m));
}

void slpa_part_det_collect_impl(slpa_ctx *ctx, uint64_t *list_dptr, int64_t *n_words, int64_t *n_marks) {
    DeviceGraph &g = ctx->g;
    WorkBuffers &wb = ctx->wb;
    cudaStream_t s = ctx->stream;
    const int64_t n = g.n, vb = ctx->v_begin, ve = ctx->v_end, nwords = (n + 31) / 32;
    wb.xlist.alloc((size_t)(2 * (ve - vb) + (n - (ve - vb)) + 1));
    wb.dcount.alloc(2);
    CUDA_TRY(cudaMemsetAsync(wb.dcount.p, 0, 2 * sizeof(unsigned long long), s));
    if (ve > vb)
        k_collect_words<<<grid_for(ve - vb, kThreads), kThreads, 0, s>>>(wb.lab_new.p, wb.lab_sent.p, vb, ve, wb.xlist.p,
                                                                         wb.dcount.p);
    CUDA_TRY(cudaGetLastError());
    unsigned long long h[2];
    CUDA_TRY(cudaMemcpyAsync(h, wb.dcount.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const int64_t nw = (int64_t)h[0];
    if (nwords > 0)
        k_collect_marks<<<grid_for(nwords, kThreads), kThreads, 0, s>>>(wb.dirty_a.p, nwords, vb, ve,
                                                                        wb.xlist.p + 2 * nw, wb.dcount.p + 1);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(h, wb.dcount.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *list_dptr = (uint64_t)(uintptr_t)wb.xlist.p;
    *n_words = nw;
    *n_marks = (int64_t)h[1];
}

int64_t slpa_part_det_apply_impl(slpa_ctx *ctx, const int32_t *recv, int64_t stride, const int64_t *counts_host,
                                 int32_t world, int32_t self) {
    DeviceGraph &g = ctx->g;
    WorkBuffers &wb = ctx->wb;
    cudaStream_t s = ctx->stream;
    const int64_t vb = ctx->v_begin, ve = ctx->v_end;
    DevBuf<int64_t> cnt;
    cnt.alloc((size_t)2 * world);
    CUDA_TRY(cudaMemcpyAsync(cnt.p, counts_host, 2 * world * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    const int64_t nwords = (g.n + 31) / 32;
    if (nwords > 0)  // this rank's marks on remote vertices went out with its list
        k_clear_remote_bits<<<grid_for(nwords, kThreads), kThreads, 0, s>>>(wb.dirty_a.p, nwords, vb, ve);
    int64_t most = 0;
    for (int r = 0; r < world; ++r) most = std::max<int64_t>(most, counts_host[2 * r] + counts_host[2 * r + 1]);
    if (most > 0) {
        const dim3 grid((unsigned)std::min<int64_t>(grid_for(most, kThreads), 4096), (unsigned)world);
        k_apply_lists<<<grid, kThreads, 0, s>>>(recv, stride, cnt.p, world, self, vb, ve, wb.lab_new.p, nullptr,
                                                wb.dirty_a.p);
    }
    wb.dcount.alloc(2);
    CUDA_TRY(cudaMemsetAsync(wb.dcount.p, 0, sizeof(unsigned long long), s));
    if (ve > vb) k_count_owned_bits<<<grid_for(ve - vb, kThreads), kThreads, 0, s>>>(wb.dirty_a.p, vb, ve, wb.dcount.p);
    CUDA_TRY(cudaGetLastError());
    unsigned long long h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, wb.dcount.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return (int64_t)h;
}

// Dense round exchange: the dirty bitmap as bytes for the host's MAX-reduce
// (the owned label words travel in the host's all-gather of lab_new).
void slpa_part_det_dense_impl(slpa_ctx *ctx) {
    const int64_t n = ctx->g.n;
    if (n > 0)
        k_dirty_bits_to_bytes<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(ctx->wb.dirty_a.p,
                                                                                   ctx->wb.dirty_bytes.p, n);
    CUDA_TRY(cudaGetLastError());
}

int64_t slpa_part_det_import_impl(slpa_ctx *ctx) {
    WorkBuffers &wb = ctx->wb;
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->g.n;
    wb.dcount.alloc(1);
    unsigned long long *cnt = wb.dcount.p;
    CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    if (n > 0) k_dirty_bytes_to_bits<<<grid_for(n, kThreads), kThreads, 0, s>>>(wb.dirty_bytes.p, wb.dirty_a.p, n, cnt);
    CUDA_TRY(cudaGetLastError());
    unsigned long long h = 0;
    CUDA_TRY(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return (int64_t)h;
}

// End of a partitioned deterministic sweep: the owned changed vertices mark
// their neighbours t <= v (possibly remote; the host MAX-reduces the flags),
// L1 is folded into L0 across the whole replica, and the flags produced by
// this sweep become the current ones.
int64_t slpa_part_det_commit_impl(slpa_ctx *ctx, const slpa_config *cfg) {
    DeviceGraph &g = ctx->g;
    WorkBuffers &wb = ctx->wb;
    cudaStream_t s = ctx->stream;
    const int64_t n = g.n;
    const SweepArgs a = make_args(ctx, cfg, 0);
    CUDA_TRY(cudaMemsetAsync(wb.counters.p + CNT_DELTA * CNT_STRIPES, 0, CNT_STRIPES * sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(wb.fbits.p, 0, (size_t)((n + 31) / 32) * sizeof(uint32_t), s));
    if (g.n_lo > 0) k_commit_lo<<<grid_for(g.n_lo, kThreads), kThreads, 0, s>>>(a, g.bin_lo.p, g.n_lo);
    if (g.n_mid > 0) k_commit_hi<<<grid_for(g.n_mid * 32, kThreads), kThreads, 0, s>>>(a, g.bin_mid.p, g.n_mid);
    if (g.n_hi > 0) k_commit_hi<<<grid_for(g.n_hi * 32, kThreads), kThreads, 0, s>>>(a, g.bin_hi.p, g.n_hi);
    if (g.n_giant > 0) commit_giants(ctx, a, s);
    if (n > 0) k_fold_all<<<grid_for(n, kThreads), kThreads, 0, s>>>(wb.lab_old.p, wb.lab_new.p, n);
    if (n > 0) k_flag_bits_to_bytes<<<grid_for((n + 3) / 4, kThreads), kThreads, 0, s>>>(wb.fbits.p, wb.flag_a.p, n);
    if (n > 0)  // every rank folded the same words: the published state is the folded one
        CUDA_TRY(cudaMemcpyAsync(wb.lab_sent.p, wb.lab_new.p, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(cudaGetLastError());
    read_counters(ctx);
    ctx->stats.sweeps += 1;
    return (int64_t)ctx->h_sum[CNT_DELTA];
}

// ====================================================================== drivers
int64_t slpa_sweep_det(slpa_ctx *ctx, const slpa_config *cfg, int pickless) {
    NvtxRange nvtx_sweep("slpa sweep (deterministic)");
    DeviceGraph &g = ctx->g;
    WorkBuffers &wb = ctx->wb;
    cudaStream_t s = ctx->stream;
    const int64_t n = g.n;
    const KernelSet ks = kernels_for(ctx, cfg, true);
    const SweepArgs a = make_args(ctx, cfg, pickless);
    SweepArgs a_r0 = a;  // round 0 of the first sweep: labels are still the ids (SweepArgs::ident)
    a_r0.ident = ctx->labels_initial && !g.has_order && ctx->lmap_mode == 0;
    CUDA_TRY(cudaMemsetAsync(wb.counters.p, 0, CNT_TOTAL * sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(wb.flag_b.p, 0, (size_t)n, s));
    for (int c = 0; c < CNT_N; ++c) ctx->h_sum[c] = 0;
    if (ctx->prof_on) CUDA_TRY(cudaMemsetAsync(wb.tbits.p, 0, (size_t)((n + 31) / 32) * sizeof(uint32_t), s));
    static const int defer = [] {
        const char *e = getenv("SLPA_DEFER");
        return e ? atoi(e) : 2;
    }();
    const int64_t nwords = (n + 31) / 32;
    // round 0: every flagged vertex, straight from the degree bins.  With
    // defer >= 2 the heavy ones (mid / hi / giant) wait for the light ones
    // to settle first -- any fair order reaches the same unique fixpoint.
    if (defer >= 2) {
        const int32_t *heavy[3] = {g.bin_hi.p, g.bin_mid.p, g.bin_giant.p};
        const int64_t nheavy[3] = {g.n_hi, g.n_mid, g.n_giant};
        for (int h = 0; h < 3; ++h)
            if (nheavy[h] > 0)
                k_defer_flagged<<<grid_for(nheavy[h], kThreads), kThreads, 0, s>>>(heavy[h], nheavy[h], wb.flag_a.p,
                                                                                  wb.dirty_b.p);
        CUDA_TRY(cudaGetLastError());
    } else {
        if (g.n_giant > 0) {
            k_iota<<<grid_for(g.n_giant, kThreads), kThreads, 0, s>>>(wb.wl_giant.p, g.n_giant);
            launch_giant(ctx, ks, a, wb.wl_giant.p, g.n_giant, 1);
        }
        launch_hi(ctx, ks, a, g.bin_hi.p, g.n_hi, 1, SLPA_PROF_EVAL_HI0);
        launch_lane(ctx, ks, 1, a, g.bin_mid.p, g.n_mid, 1, SLPA_PROF_EVAL_MID0);
    }
    // Round 0, light vertices: only the flagged entries of the degree-ordered
    // bin.  After sweep 0 a minority is flagged; launching the whole bin would
    // leave most lanes of every warp idle while the few flagged ones run the
    // full evaluation.
    if (g.n_lo > 0 && round0_compact()) {
        unsigned long long *c0 = wb.counters.p + CNT_LO * CNT_STRIPES;
        timed_launch(ctx, SLPA_PROF_COMPACT, 1, [&] {
            k_filter_flags<<<grid_for(g.n_lo, kThreads), kThreads, 0, s>>>(g.bin_lo.p, g.n_lo, wb.flag_a.p,
                                                                          wb.wl_lo.p, c0);
            CUDA_TRY(cudaGetLastError());
        });
        unsigned long long nf = 0;
        CUDA_TRY(cudaMemcpyAsync(&nf, c0, sizeof(nf), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        launch_lane(ctx, ks, 0, a_r0, wb.wl_lo.p, (int64_t)nf, 1, SLPA_PROF_EVAL_LO0);
    } else {
        launch_lane(ctx, ks, 0, a_r0, g.bin_lo.p, g.n_lo, 1, SLPA_PROF_EVAL_LO0);
    }
    ctx->labels_initial = 0;
    int64_t rounds = 1;
    unsigned long long evals0 = 0, arcs0 = 0;
    bool first = true;
    unsigned long long *cur_lo = wb.counters.p + CNT_LO * CNT_STRIPES, *cur_mid = wb.counters.p + CNT_MID * CNT_STRIPES,
                       *cur_hi = wb.counters.p + CNT_HI * CNT_STRIPES,
                       *cur_giant = wb.counters.p + CNT_GIANT * CNT_STRIPES;
    bool pend_any = defer != 0;
    // Asynchronous giants (default with deferral and the bitmap scan): a giant
    // batch runs on the priority stream while the rounds go on; its dependant
    // marks go to dirty_g and are OR-ed into the round bitmap once the batch
    // has finished, marks for giants wait in dirty_gp, and at most one batch
    // is in flight (its gather buffer).  A giant that read a label which
    // changed later is marked by that change like any other vertex, so the
    // fixpoint -- the sequential sweep -- is unchanged; the rounds just no
    // longer wait for the giants' long chunk chains.
    const bool agiant = defer >= 2 && scan_mode() && g.n_giant > 0 && !ctx->prof_on && giant_async_mode();
    bool g_inflight = false;
    int64_t g_pending = 0;
    SweepArgs ag = a;
    if (agiant) {
        ag.dirty_next = wb.dirty_g.p;
        CUDA_TRY(cudaMemsetAsync(wb.dirty_g.p, 0, (size_t)nwords * sizeof(uint32_t), s));
        CUDA_TRY(cudaMemsetAsync(wb.dirty_gp.p, 0, (size_t)nwords * sizeof(uint32_t), s));
        g_pending = g.n_giant;  // round 0: flagged giants sit in dirty_b, moved below
        k_move_class<<<grid_for(g.n_giant, kThreads), kThreads, 0, s>>>(g.bin_giant.p, g.n_giant, wb.dirty_b.p,
                                                                       wb.dirty_gp.p);
        CUDA_TRY(cudaGetLastError());
    }
    for (;;) {
        NvtxRange nvtx_round("slpa round");
        if (agiant) {
            if (g_inflight && cudaEventQuery(ctx->gev1) == cudaSuccess) {
                k_or_clear<<<grid_for(nwords, kThreads), kThreads, 0, s>>>(wb.dirty_g.p, wb.dirty_a.p, nwords);
                CUDA_TRY(cudaGetLastError());
                g_inflight = false;
                ctx->giant_pending = 0;
            }
        } else {
            giant_join(ctx);
        }
        CUDA_TRY(cudaMemsetAsync(cur_lo, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(cur_mid, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(cur_hi, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(cur_giant, 0, sizeof(unsigned long long), s));
        const bool bitmap_scan = defer && scan_mode();
        timed_launch(ctx, SLPA_PROF_COMPACT, bitmap_scan ? 1 : 4, [&] {
            if (bitmap_scan) {
                k_scan_dirty<<<grid_for(nwords, kThreads), kThreads, 0, s>>>(
                    wb.dirty_a.p, wb.dirty_b.p, g.cls.p, nwords, wb.wl_lo.p, cur_lo, agiant ? wb.dirty_gp.p : nullptr,
                    wb.counters.p + CNT_GPEND * CNT_STRIPES);
                return;
            }
            launch_filter(s, g.bin_lo.p, g.n_lo, wb.dirty_a.p, wb.wl_lo.p, cur_lo);
            if (defer) {
                const int32_t *heavy[3] = {g.bin_hi.p, g.bin_mid.p, g.bin_giant.p};
                const int64_t nheavy[3] = {g.n_hi, g.n_mid, g.n_giant};
                for (int h = 0; h < 3; ++h)
                    if (nheavy[h] > 0)
                        k_defer_dirty<<<grid_for(nheavy[h], kThreads), kThreads, 0, s>>>(heavy[h], nheavy[h],
                                                                                        wb.dirty_a.p, wb.dirty_b.p);
            } else {
                launch_filter(s, g.bin_hi.p, g.n_hi, wb.dirty_a.p, wb.wl_hi.p, cur_hi);
                launch_filter(s, g.bin_mid.p, g.n_mid, wb.dirty_a.p, wb.wl_mid.p, cur_mid);
                launch_filter(s, g.bin_giant.p, g.n_giant, wb.dirty_a.p, wb.wl_giant.p, cur_giant, 1);
            }
            CUDA_TRY(cudaGetLastError());
        });
        read_counters(ctx);
        // (rows of at most 8 arcs stream unaligned, so their order matters little)
        if (bitmap_scan && (int64_t)ctx->h_sum[CNT_LO] > scan_sort_min() && g.lo_max_deg > 8) {
            // large round: the degree-ordered worklist keeps the lanes of a warp on similar row lengths
            CUDA_TRY(cudaMemsetAsync(cur_lo, 0, sizeof(unsigned long long), s));
            timed_launch(ctx, SLPA_PROF_COMPACT, 1, [&] {
                launch_filter(s, g.bin_lo.p, g.n_lo, wb.dirty_a.p, wb.wl_lo.p, cur_lo);
                CUDA_TRY(cudaGetLastError());
            });
        }
        CUDA_TRY(cudaMemsetAsync(wb.dirty_a.p, 0, (size_t)nwords * sizeof(uint32_t), s));
        if (first) {
            evals0 = ctx->h_sum[CNT_EVALS] + ctx->h_sum[CNT_EVALS_HI];
            arcs0 = ctx->h_sum[CNT_ARCS] + ctx->h_sum[CNT_ARCS_HI];
            first = false;
        }
        int64_t nlo = (int64_t)ctx->h_sum[CNT_LO], nmid = (int64_t)ctx->h_sum[CNT_MID],
                nhi = (int64_t)ctx->h_sum[CNT_HI], ngiant = (int64_t)ctx->h_sum[CNT_GIANT];
        if (agiant) g_pending += (int64_t)ctx->h_sum[CNT_GPEND];
        CUDA_TRY(cudaMemsetAsync(wb.counters.p + CNT_GPEND * CNT_STRIPES, 0, sizeof(unsigned long long), s));
        const bool quiet = nlo <= defer_min(g.n_lo);
        const bool launch_g = agiant && quiet && !g_inflight && g_pending > 0;
        if (defer && quiet && (pend_any || launch_g)) {  // light vertices (nearly) quiet: run the pending heavy ones
            timed_launch(ctx, SLPA_PROF_COMPACT, 3, [&] {
                if (pend_any) {
                    launch_filter(s, g.bin_hi.p, g.n_hi, wb.dirty_b.p, wb.wl_hi.p, cur_hi);
                    launch_filter(s, g.bin_mid.p, g.n_mid, wb.dirty_b.p, wb.wl_mid.p, cur_mid);
                    if (!agiant) launch_filter(s, g.bin_giant.p, g.n_giant, wb.dirty_b.p, wb.wl_giant.p, cur_giant, 1);
                }
                if (launch_g) launch_filter(s, g.bin_giant.p, g.n_giant, wb.dirty_gp.p, wb.wl_giant.p, cur_giant, 1);
                CUDA_TRY(cudaGetLastError());
            });
            if (pend_any) CUDA_TRY(cudaMemsetAsync(wb.dirty_b.p, 0, (size_t)nwords * sizeof(uint32_t), s));
            if (launch_g) {
                CUDA_TRY(cudaMemsetAsync(wb.dirty_gp.p, 0, (size_t)nwords * sizeof(uint32_t), s));
                g_pending = 0;
            }
            read_counters(ctx);
            nmid = (int64_t)ctx->h_sum[CNT_MID];
            nhi = (int64_t)ctx->h_sum[CNT_HI];
            ngiant = (int64_t)ctx->h_sum[CNT_GIANT];
        }
        if (trace_rounds()) {
            static auto t_prev = std::chrono::steady_clock::now();
            const auto t_now = std::chrono::steady_clock::now();
            fprintf(stderr, "[slpa] sweep round %lld: lo %lld mid %lld hi %lld giant %lld  (+%.0f us)\n",
                    (long long)rounds, (long long)nlo, (long long)nmid, (long long)nhi, (long long)ngiant,
                    std::chrono::duration<double, std::micro>(t_now - t_prev).count());
            t_prev = t_now;
        }
        if (nlo == 0 && nmid == 0 && nhi == 0 && ngiant == 0) {
            if (!agiant || (!g_inflight && g_pending == 0)) break;
            if (g_inflight) {  // only the giant batch is left: wait for it, merge its marks
                CUDA_TRY(cudaEventSynchronize(ctx->gev1));
                k_or_clear<<<grid_for(nwords, kThreads), kThreads, 0, s>>>(wb.dirty_g.p, wb.dirty_a.p, nwords);
                CUDA_TRY(cudaGetLastError());
                g_inflight = false;
                ctx->giant_pending = 0;
            }
            pend_any = true;  // the merged marks may include deferred heavy vertices
            continue;
        }
        pend_any = defer != 0;
        if (agiant) {
            if (ngiant > 0) {
                launch_giant(ctx, ks, ag, wb.wl_giant.p, ngiant, 0);
                g_inflight = true;
            }
        } else {
            launch_giant(ctx, ks, a, wb.wl_giant.p, ngiant, 0);
        }
        launch_hi(ctx, ks, a, wb.wl_hi.p, nhi, 0, SLPA_PROF_EVAL_HIK);
        launch_lane(ctx, ks, 0, a, wb.wl_lo.p, nlo, 0, SLPA_PROF_EVAL_LOK, true);
        launch_lane(ctx, ks, 1, a, wb.wl_mid.p, nmid, 0, SLPA_PROF_EVAL_MIDK);
        ++rounds;
    }
    giant_join(ctx);
    const unsigned long long evals = ctx->h_sum[CNT_EVALS] + ctx->h_sum[CNT_EVALS_HI];
    const unsigned long long arcs = ctx->h_sum[CNT_ARCS] + ctx->h_sum[CNT_ARCS_HI];
    NvtxRange nvtx_commit("slpa commit");
    // commit: L0 <- L1, delta, next-sweep flags pushed from the changed rows
    const int64_t fwords = (n + 31) / 32;
    CUDA_TRY(cudaMemsetAsync(wb.fbits.p, 0, (size_t)fwords * sizeof(uint32_t), s));
    timed_launch(ctx, SLPA_PROF_COMMIT, g.n_giant > 0 ? 6 : 5, [&] {
        if (g.n_lo > 0) {
            if (commit_pos_mode()) k_commit_lo_pos<<<grid_for(n, kThreads), kThreads, 0, s>>>(a, n);
            else k_commit_lo<<<grid_for(g.n_lo, kThreads), kThreads, 0, s>>>(a, g.bin_lo.p, g.n_lo);
        }
        if (g.n_mid > 0) k_commit_hi<<<grid_for(g.n_mid * 32, kThreads), kThreads, 0, s>>>(a, g.bin_mid.p, g.n_mid);
        if (g.n_hi > 0) k_commit_hi<<<grid_for(g.n_hi * 32, kThreads), kThreads, 0, s>>>(a, g.bin_hi.p, g.n_hi);
        if (g.n_giant > 0) commit_giants(ctx, a, s);
        if (n > 0) k_flag_bits_to_bytes<<<grid_for((n + 3) / 4, kThreads), kThreads, 0, s>>>(wb.fbits.p, wb.flag_b.p, n);
        CUDA_TRY(cudaGetLastError());
    });
    read_counters(ctx);
    if (trace_rounds() >= 3 && !timeline().empty()) {
        CUDA_TRY(cudaDeviceSynchronize());
        const char *names[] = {"lo0", "mid0", "hi0", "lo", "mid", "hi", "compact", "commit", "other", "giant"};
        cudaEvent_t base = timeline().front().e0;
        for (const TimelineEv &ev : timeline()) {
            float t0 = 0.f, t1 = 0.f;
            cudaEventElapsedTime(&t0, base, ev.e0);
            cudaEventElapsedTime(&t1, base, ev.e1);
            fprintf(stderr, "[slpa] tl %-8s %s %9.1f %9.1f %8.1f\n", ev.cls >= 0 && ev.cls < 10 ? names[ev.cls] : "?",
                    ev.giant ? "G" : "M", 1000.f * t0, 1000.f * t1, 1000.f * (t1 - t0));
        }
        for (const TimelineEv &ev : timeline()) {
            cudaEventDestroy(ev.e0);
            cudaEventDestroy(ev.e1);
        }
        timeline().clear();
        cudaGetLastError();
    }
    std::swap(wb.flag_a, wb.flag_b);
    ctx->stats.rounds += rounds;
    ctx->stats.vertex_evals += (int64_t)evals;
    ctx->stats.arc_reads += (int64_t)arcs;
    if (ctx->prof_on && n > 0) {  // the sequential sweep's processed set, from the turn bitmap
        wb.dcount.alloc(2);
        CUDA_TRY(cudaMemsetAsync(wb.dcount.p, 0, 2 * sizeof(unsigned long long), s));
        const int64_t nw = (n + 31) / 32;
        k_count_turns<<<grid_for(nw, kThreads), kThreads, 0, s>>>(wb.tbits.p, g.off(), wb.flag_b.p /* F0, swapped above */, n, wb.dcount.p);
        CUDA_TRY(cudaGetLastError());
        unsigned long long h[2] = {0, 0};
        CUDA_TRY(cudaMemcpyAsync(h, wb.dcount.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        ctx->stats.first_evals += (int64_t)h[0];
        ctx->stats.first_arcs += (int64_t)h[1];
    }
    (void)evals0;
    (void)arcs0;
    return (int64_t)ctx->h_sum[CNT_DELTA];
}

int64_t slpa_sweep_async(slpa_ctx *ctx, const slpa_config *cfg, int pickless) {
    NvtxRange nvtx_sweep("slpa sweep (async)");
    DeviceGraph &g = ctx->g;
    WorkBuffers &wb = ctx->wb;
    cudaStream_t s = ctx->stream;
    const KernelSet ks = kernels_for(ctx, cfg, false);
    const SweepArgs a = make_args(ctx, cfg, pickless);
    CUDA_TRY(cudaMemsetAsync(wb.counters.p, 0, CNT_TOTAL * sizeof(unsigned long long), s));
    for (int c = 0; c < CNT_N; ++c) ctx->h_sum[c] = 0;
    // Higher-degree vertices first: they carry most arcs and the tail.
    if (g.n_giant > 0) {
        k_iota<<<grid_for(g.n_giant, kThreads), kThreads, 0, s>>>(wb.wl_giant.p, g.n_giant);
        launch_giant(ctx, ks, a, wb.wl_giant.p, g.n_giant, 1);
    }
    launch_hi(ctx, ks, a, g.bin_hi.p, g.n_hi, 1, SLPA_PROF_EVAL_HI0);
    launch_lane(ctx, ks, 1, a, g.bin_mid.p, g.n_mid, 1, SLPA_PROF_EVAL_MID0);
    launch_lane(ctx, ks, 0, a, g.bin_lo.p, g.n_lo, 1, SLPA_PROF_EVAL_LO0);
    giant_join(ctx);
    if (!ctx->part) {  // partitioned: remote entries hold outgoing marks, cleared after the exchange
        timed_launch(ctx, SLPA_PROF_OTHER, 1, [&] {
            k_clear_isolated_flags<<<grid_for(g.n, kThreads), kThreads, 0, s>>>(wb.flag_a.p, g.cls.p, g.n);
            CUDA_TRY(cudaGetLastError());
        });
    }
    read_counters(ctx);
    const int64_t ev = (int64_t)(ctx->h_sum[CNT_EVALS] + ctx->h_sum[CNT_EVALS_HI]);
    const int64_t ar = (int64_t)(ctx->h_sum[CNT_ARCS] + ctx->h_sum[CNT_ARCS_HI]);
    ctx->labels_initial = 0;
    ctx->stats.rounds += 1;
    ctx->stats.vertex_evals += ev;
    ctx->stats.arc_reads += ar;
    ctx->stats.first_evals += ev;
    ctx->stats.first_arcs += ar;
    return (int64_t)ctx->h_sum[CNT_DELTA];
}

// ------------------------------------------------------------------ caller label values
// The kernels keep labels in 31 bits (bit 31 of lab_new is the changed
// flag).  Caller labels (lpa_move, a hook that edits the live array) may be
// any int32 (lpa.py:227-259).  The sweep only compares labels (equality,
// order for pick-less sweeps and ties) and never creates new values, so an
// order-preserving map of the label set into [0, 2^31) is exact: a shift by
// the minimum when the span fits, else the rank in sorted(labels + {0}).
// The sketches start every key as "label 0" (sketch.py:38) -- its image
// under the map is SweepArgs::zkey.  Labels go back through the inverse.
__global__ void k_minmax_i32(const int32_t *__restrict__ x, int64_t n, int *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int lo = INT_MAX, hi = INT_MIN;
    if (i < n) lo = hi = x[i];
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&out[0], lo);
        atomicMax(&out[1], hi);
    }
}
__global__ void k_shift_i32(const int32_t *__restrict__ in, int32_t *__restrict__ out, int64_t n, int64_t d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)((int64_t)in[i] + d);
}
__global__ void k_rank_i32(int32_t *__restrict__ x, int64_t n, const int32_t *__restrict__ table, int64_t nt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t v = x[i];
    int64_t lo = 0, hi = nt - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(&table[mid]) < v) lo = mid + 1;
        else hi = mid;
    }
    x[i] = (int32_t)lo;
}
__global__ void k_unrank_i32(const int32_t *__restrict__ in, int32_t *__restrict__ out, int64_t n,
                             const int32_t *__restrict__ table) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __ldg(&table[in[i]]);
}

// lab_old (by position) holds raw caller labels: map them in place.
void map_caller_labels(slpa_ctx *ctx, const int32_t *host_by_id) {
    const int64_t n = ctx->g.n;
    cudaStream_t s = ctx->stream;
    ctx->lmap_mode = 0;
    ctx->lmap_shift = 0;
    ctx->zkey = 0;
    WorkBuffers &wb = ctx->wb;
    wb.dcount.alloc(2);
    int *mm = reinterpret_cast<int *>(wb.dcount.p);
    const int init[2] = {INT_MAX, INT_MIN};
    CUDA_TRY(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_minmax_i32<<<grid_for(n, kThreads), kThreads, 0, s>>>(wb.lab_old.p, n, mm);
    CUDA_TRY(cudaGetLastError());
    int h[2];
    CUDA_TRY(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (h[0] >= 0) return;  // the common case: labels are already non-negative
    const int64_t lo = h[0], hi = std::max<int64_t>(h[1], 0);
    if (hi - lo < (int64_t)SLPA_LMASK) {  // shift by the minimum
        ctx->lmap_mode = 1;
        ctx->lmap_shift = lo;
        ctx->zkey = (int32_t)(-lo);
        k_shift_i32<<<grid_for(n, kThreads), kThreads, 0, s>>>(wb.lab_old.p, wb.lab_old.p, n, -lo);
        CUDA_TRY(cudaGetLastError());
        return;
    }
    // rank in the sorted label set (plus 0, so label 0 has an image)
    std::vector<int32_t> t(host_by_id, host_by_id + n);
    t.push_back(0);
    std::sort(t.begin(), t.end());
    t.erase(std::unique(t.begin(), t.end()), t.end());
    ctx->lmap_table.alloc(t.size());
    CUDA_TRY(cudaMemcpyAsync(ctx->lmap_table.p, t.data(), t.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    ctx->lmap_n = (int64_t)t.size();
    ctx->lmap_mode = 2;
    ctx->zkey = (int32_t)(std::lower_bound(t.begin(), t.end(), 0) - t.begin());
    k_rank_i32<<<grid_for(n, kThreads), kThreads, 0, s>>>(wb.lab_old.p, n, ctx->lmap_table.p, ctx->lmap_n);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));  // t is freed on return
}

void slpa_init_labels(slpa_ctx *ctx) {
    ctx->labels_initial = 1;
    ctx->lmap_mode = 0;
    ctx->lmap_shift = 0;
    ctx->zkey = 0;
    const int64_t n = ctx->g.n;
    if (n == 0) return;
    k_init_labels<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(
        ctx->wb.lab_old.p, ctx->wb.lab_new.p, ctx->wb.flag_a.p, ctx->g.has_order ? ctx->g.ids.p : nullptr, n);
    CUDA_TRY(cudaGetLastError());
}

void slpa_labels_to_host(slpa_ctx *ctx, int32_t *host) {
    const int64_t n = ctx->g.n;
    if (n == 0) return;
    const int32_t *src = ctx->wb.lab_old.p;
    DevBuf<int32_t> unmapped;
    if (ctx->lmap_mode) {  // back to the caller's label values
        unmapped.alloc(n);
        if (ctx->lmap_mode == 1)
            k_shift_i32<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(src, unmapped.p, n, ctx->lmap_shift);
        else
            k_unrank_i32<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(src, unmapped.p, n, ctx->lmap_table.p);
        CUDA_TRY(cudaGetLastError());
        src = unmapped.p;
    }
    if (ctx->g.has_order) {
        k_pos_to_id_i32<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(src, ctx->wb.io_labels.p, ctx->g.ids.p, n);
        CUDA_TRY(cudaGetLastError());
        src = ctx->wb.io_labels.p;
    }
    // through a pinned staging buffer (full-speed DMA), then a parallel host copy
    if (ctx->h_stage_n < n) {
        if (ctx->h_stage) CUDA_TRY(cudaFreeHost(ctx->h_stage));
        ctx->h_stage = nullptr;
        CUDA_TRY(cudaMallocHost((void **)&ctx->h_stage, (size_t)n * sizeof(int32_t)));
        ctx->h_stage_n = n;
    }
    CUDA_TRY(cudaMemcpyAsync(ctx->h_stage, src, n * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    const int nt = n >= (1 << 22) ? 8 : 1;
    if (nt == 1) {
        std::memcpy(host, ctx->h_stage, (size_t)n * sizeof(int32_t));
    } else {
        std::vector<std::thread> th;
        const int64_t per = (n + nt - 1) / nt;
        for (int i = 0; i < nt; ++i) {
            const int64_t b = i * per, e = std::min<int64_t>(n, b + per);
            if (b < e)
                th.emplace_back([=] { std::memcpy(host + b, ctx->h_stage + b, (size_t)(e - b) * sizeof(int32_t)); });
        }
        for (auto &t : th) t.join();
    }
}

void slpa_labels_from_host(slpa_ctx *ctx, const int32_t *host) {
    const int64_t n = ctx->g.n;
    if (n == 0) return;
    if (ctx->g.has_order) {
        CUDA_TRY(cudaMemcpyAsync(ctx->wb.io_labels.p, host, n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        k_id_to_pos_i32<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(ctx->wb.io_labels.p, ctx->wb.lab_old.p,
                                                                              ctx->g.ids.p, n);
    } else {
        CUDA_TRY(cudaMemcpyAsync(ctx->wb.lab_old.p, host, n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    }
    map_caller_labels(ctx, host);
    ctx->labels_initial = 0;
    k_sync_lab_new<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(ctx->wb.lab_old.p, ctx->wb.lab_new.p, n);
    CUDA_TRY(cudaGetLastError());
}

void slpa_flags_to_host(slpa_ctx *ctx, uint8_t *host) {
    const int64_t n = ctx->g.n;
    if (n == 0) return;
    const uint8_t *src = ctx->wb.flag_a.p;
    if (ctx->g.has_order) {
        k_pos_to_id_u8<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(src, ctx->wb.io_flags.p, ctx->g.ids.p, n);
        CUDA_TRY(cudaGetLastError());
        src = ctx->wb.io_flags.p;
    }
    CUDA_TRY(cudaMemcpyAsync(host, src, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
}

void slpa_flags_from_host(slpa_ctx *ctx, const uint8_t *host) {
    const int64_t n = ctx->g.n;
    if (n == 0) return;
    if (ctx->g.has_order) {
        CUDA_TRY(cudaMemcpyAsync(ctx->wb.io_flags.p, host, (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
        k_id_to_pos_u8<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(ctx->wb.io_flags.p, ctx->wb.flag_a.p,
                                                                             ctx->g.ids.p, n);
    } else {
        CUDA_TRY(cudaMemcpyAsync(ctx->wb.flag_a.p, host, (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
        k_norm_flags<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(ctx->wb.flag_a.p, n);
    }
    CUDA_TRY(cudaGetLastError());
}

void slpa_permute_id_to_pos(slpa_ctx *ctx, const int32_t *d_by_id, int32_t *d_by_pos) {
    const int64_t n = ctx->g.n;
    if (n == 0) return;
    k_id_to_pos_i32<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(d_by_id, d_by_pos, ctx->g.ids.p, n);
    CUDA_TRY(cudaGetLastError());
}
