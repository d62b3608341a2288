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
#include <cstdlib>
#include "slpa_sketch.cuh"
#include "slpa_internal.cuh"

namespace {

constexpr int kThreads = 256;

// ------------------------------------------------------------------ label reads
// Deterministic mode: neighbour t of v (positions).  Lower neighbours give
// L1 (speculative, possibly written this round -> L2 load), higher ones L0.
// The hot array is lab_new (L1 | changed<<31); a higher neighbour's L0 is
// fetched from lab_old only when its changed bit is set, so most gathers
// touch one n*4-byte array (L2-resident at RMAT scale 24).
__device__ __forceinline__ int32_t det_label(const SweepArgs &a, int32_t t, int32_t v, bool &lower_changed) {
    const uint32_t L = __ldcg(&a.lab_new[t]);
    if (t < v) {
        lower_changed |= (L >> 31) != 0;
        return (int32_t)(L & SLPA_LMASK);
    }
    return (L >> 31) ? __ldg(&a.lab_old[t]) : (int32_t)L;
}

__device__ __forceinline__ int32_t async_label(const SweepArgs &a, int32_t t) { return __ldcg(&a.lab_old[t]); }

// CSR streams (read once per sweep) are loaded with an L2 evict-first policy
// so they do not push the label array out of L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t *ptr, uint64_t pol) {
    int32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ float ld_stream(const float *ptr, uint64_t pol) {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_stream(const double *ptr, uint64_t pol) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(ptr), "l"(pol));
    return r;
}

template <class W>
__device__ __forceinline__ double arc_weight(const SweepArgs &a, int64_t e) {
    return (double)__ldg(reinterpret_cast<const W *>(a.w) + e);
}

// T for an asymmetric graph: some lower in-neighbour changed.
__device__ __forceinline__ bool lower_in_changed(const SweepArgs &a, int32_t v) {
    for (int64_t e = a.roff[v]; e < a.roff[v + 1]; ++e) {
        int32_t u = a.rsrc[e];
        if (u < v && (__ldcg(&a.lab_new[u]) >> 31)) return true;
    }
    return false;
}

__device__ __forceinline__ void mark_dirty(uint32_t *bm, int32_t t) { atomicOr(&bm[t >> 5], 1u << (t & 31)); }

// Re-queue v's higher-positioned dependants (readers of v's label and
// vertices whose turn depends on v's changed bit).
__device__ __forceinline__ void mark_dependants(const SweepArgs &a, int32_t v, int64_t lo, int64_t hi, int start,
                                                int stride) {
    for (int64_t e = lo + start; e < hi; e += stride) {
        int32_t t = __ldg(&a.tgt[e]);
        if (t > v) mark_dirty(a.dirty_next, t);
    }
    if (!a.symmetric) {
        for (int64_t e = a.roff[v] + start; e < a.roff[v + 1]; e += stride) {
            int32_t u = a.rsrc[e];
            if (u > v) mark_dirty(a.dirty_next, u);
        }
    }
}

// Counters are striped over CNT_STRIPES slots (by warp) so that per-warp
// atomics do not serialise on one L2 address; the host sums the stripes.
__device__ __forceinline__ int stripe() {
    return (int)((((unsigned)blockIdx.x * blockDim.x + threadIdx.x) >> 5) & (CNT_STRIPES - 1));
}
__device__ __forceinline__ void ctr_add(unsigned long long *ctr, int which, unsigned long long x) {
    atomicAdd(&ctr[which * CNT_STRIPES + stripe()], x);
}

// Warp-aggregated counter update; every lane of the warp must call it.
__device__ __forceinline__ void warp_count(unsigned long long *ctr, unsigned long long evals,
                                           unsigned long long arcs, unsigned long long delta) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        evals += __shfl_xor_sync(0xffffffffu, evals, o);
        arcs += __shfl_xor_sync(0xffffffffu, arcs, o);
        delta += __shfl_xor_sync(0xffffffffu, delta, o);
    }
    if ((threadIdx.x & 31) == 0) {
        const int s = stripe();
        if (evals) atomicAdd(&ctr[CNT_EVALS * CNT_STRIPES + s], evals);
        if (arcs) atomicAdd(&ctr[CNT_ARCS * CNT_STRIPES + s], arcs);
        if (delta) atomicAdd(&ctr[CNT_DELTA * CNT_STRIPES + s], delta);
    }
}

// Finish one deterministic evaluation (thread-per-vertex flavour).
__device__ __forceinline__ void det_commit_output(const SweepArgs &a, int32_t v, int32_t cur, int32_t cand, bool T,
                                                  int64_t lo, int64_t hi) {
    bool chg = T && cand != cur && (!a.pickless || cand < cur);
    uint32_t nw = chg ? ((uint32_t)cand | SLPA_CHG) : (uint32_t)cur;
    uint32_t ow = __ldcg(&a.lab_new[v]);
    if (nw != ow) {
        __stcg(&a.lab_new[v], nw);
        mark_dependants(a, v, lo, hi, 0, 1);
    }
}

__device__ __forceinline__ void async_commit_output(const SweepArgs &a, int32_t v, int32_t cur, int32_t cand,
                                                    int64_t lo, int64_t hi, unsigned long long &delta) {
    if (cand != cur && (!a.pickless || cand < cur)) {
        __stcg(&a.lab_old[v], cand);
        delta = 1;
        for (int64_t e = lo; e < hi; ++e) a.flag_cur[__ldg(&a.tgt[e])] = 1;
    }
}

// Finish one evaluation in a warp-per-vertex kernel (all lanes call it with
// warp-uniform arguments except lower_changed).
template <bool DET>
__device__ __forceinline__ void warp_hi_finish(const SweepArgs &a, int32_t v, int32_t cur, int32_t cand, uint8_t f0,
                                               bool lower_changed, int64_t lo, int64_t hi, int lane) {
    if (DET) {
        bool T = f0 != 0;
        if (!T) T = a.symmetric ? __any_sync(0xffffffffu, lower_changed) : lower_in_changed(a, v);
        bool chg = T && cand != cur && (!a.pickless || cand < cur);
        uint32_t nw = chg ? ((uint32_t)cand | SLPA_CHG) : (uint32_t)cur;
        uint32_t ow = __ldcg(&a.lab_new[v]);
        __syncwarp();
        if (nw != ow) {
            if (lane == 0) __stcg(&a.lab_new[v], nw);
            mark_dependants(a, v, lo, hi, lane, 32);
        }
        if (lane == 0) {
            ctr_add(a.counters, CNT_EVALS_HI, 1ull);
            ctr_add(a.counters, CNT_ARCS_HI, (unsigned long long)(hi - lo));
        }
    } else {
        if (cand != cur && (!a.pickless || cand < cur)) {
            if (lane == 0) {
                __stcg(&a.lab_old[v], cand);
                ctr_add(a.counters, CNT_DELTA, 1ull);
            }
            for (int64_t e = lo + lane; e < hi; e += 32) a.flag_cur[__ldg(&a.tgt[e])] = 1;
        }
        if (lane == 0) {
            ctr_add(a.counters, CNT_EVALS_HI, 1ull);
            ctr_add(a.counters, CNT_ARCS_HI, (unsigned long long)(hi - lo));
        }
    }
}

// ================================================================== window staging
// A warp runs 32 sequential streams (one per lane): 32 rows (low degree) or
// the 32 chunks of one vertex (high degree).  For each window of S steps the
// warp stages the next <= S arcs of every stream into a padded shared tile
// [lane][step] -- the concatenated window is loaded with consecutive lanes on
// consecutive arcs (coalesced targets / weights, 32 independent label
// gathers per instruction) -- then every lane replays its own S steps in
// order.  Self-arcs are staged with weight 0 (weights are > 0).
constexpr int kWinWarps = 4;
constexpr int kWinThreads = kWinWarps * 32;

template <class W>
struct WinS {
    static constexpr int S = sizeof(W) == 4 ? 32 : 16;
};

template <class W, bool DET, bool GRID, class Consume>
__device__ __forceinline__ void window_streams(const SweepArgs &a, uint32_t (*s_lab)[WinS<W>::S + 1],
                                               W (*s_w)[WinS<W>::S + 1], int lane, int64_t start, int64_t len,
                                               int32_t sv, bool &lower_changed, Consume &&consume) {
    constexpr int S = WinS<W>::S;
    constexpr int G = 8;  // staging iterations in flight per lane
    const W *__restrict__ wts = reinterpret_cast<const W *>(a.w);
    const uint64_t pol = policy_evict_first();
    int64_t maxlen = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        int64_t x = __shfl_xor_sync(0xffffffffu, maxlen, o);
        maxlen = x > maxlen ? x : maxlen;
    }
    for (int64_t s0 = 0; s0 < maxlen; s0 += S) {
        const int64_t rem = len - s0;
        const int seg = rem <= 0 ? 0 : (rem >= S ? S : (int)rem);
        int excl = 0, total = 0, iters;
        if (GRID) {
            // stream j's window is staged by iteration j, lane = step (coalesced)
            iters = 32;
        } else {
            int incl = seg;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int x = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += x;
            }
            excl = incl - seg;
            total = __shfl_sync(0xffffffffu, incl, 31);
            iters = (total + 31) >> 5;
        }
        for (int j0 = 0; j0 < iters; j0 += G) {
            int32_t t[G], ov[G];
            W w[G];
            int own[G], stp[G];
            bool ok[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const int j = j0 + u;
                int o, sp;
                bool valid;
                if (GRID) {
                    o = j & 31;
                    sp = lane;
                    const int sj = __shfl_sync(0xffffffffu, seg, o);
                    valid = j < 32 && lane < sj;
                } else {
                    const int va = j * 32 + lane;
                    o = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        int ex = __shfl_sync(0xffffffffu, excl, (o + step) & 31);
                        if (o + step < 32 && ex <= va) o += step;
                    }
                    sp = va - __shfl_sync(0xffffffffu, excl, o);
                    valid = va < total;
                }
                const int64_t o_start = __shfl_sync(0xffffffffu, start, o);
                ov[u] = __shfl_sync(0xffffffffu, sv, o);
                own[u] = o;
                stp[u] = sp;
                ok[u] = valid;
                if (valid) {
                    const int64_t e = o_start + s0 + sp;
                    t[u] = ld_stream(&a.tgt[e], pol);
                    w[u] = ld_stream(&wts[e], pol);
                } else {
                    t[u] = 0;
                    w[u] = (W)0;
                }
            }
            uint32_t L[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                L[u] = 0;
                if (ok[u] && t[u] != ov[u]) L[u] = DET ? __ldcg(&a.lab_new[t[u]]) : (uint32_t)__ldcg(&a.lab_old[t[u]]);
            }
            if (DET) {  // higher neighbour that changed this sweep: its L0
#pragma unroll
                for (int u = 0; u < G; ++u)
                    if (ok[u] && t[u] > ov[u] && (L[u] >> 31)) L[u] = (uint32_t)__ldg(&a.lab_old[t[u]]);
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
                if (ok[u]) {
                    s_lab[own[u]][stp[u]] = L[u];
                    s_w[own[u]][stp[u]] = (t[u] == ov[u]) ? (W)0 : w[u];
                }
            }
        }
        __syncwarp();
#pragma unroll 4
        for (int x = 0; x < seg; ++x) {
            const W w = s_w[lane][x];
            const uint32_t L = s_lab[lane][x];
            const bool valid = w != (W)0;
            lower_changed |= valid && (L >> 31) != 0;
            consume(s0 + x, valid, (int32_t)(L & SLPA_LMASK), w);
        }
        __syncwarp();
    }
}

// ================================================================== lane kernels
// One lane per vertex.  Lane outputs are written per lane; adjacency walks
// for changed vertices (dependant marks in deterministic mode, neighbour
// flags in async mode) are done by the whole warp, one changed lane at a
// time, so they are coalesced instead of 32 divergent row loops.
template <bool DET>
__device__ __forceinline__ void lane_finish(const SweepArgs &a, bool go, int32_t v, int32_t cur, int32_t cand,
                                            bool T, int64_t lo, int64_t deg, unsigned long long &n_delta) {
    const int lane = threadIdx.x & 31;
    bool walk = false;
    if (go) {
        if (DET) {
            const bool chg = T && cand != cur && (!a.pickless || cand < cur);
            const uint32_t nw = chg ? ((uint32_t)cand | SLPA_CHG) : (uint32_t)cur;
            if (nw != __ldcg(&a.lab_new[v])) {
                __stcg(&a.lab_new[v], nw);
                walk = true;
            }
        } else if (cand != cur && (!a.pickless || cand < cur)) {
            __stcg(&a.lab_old[v], cand);
            n_delta = 1;
            walk = true;
        }
    }
    unsigned m = __ballot_sync(0xffffffffu, walk);
    while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const int32_t vj = __shfl_sync(0xffffffffu, v, j);
        const int64_t lj = __shfl_sync(0xffffffffu, lo, j);
        const int64_t hj = lj + __shfl_sync(0xffffffffu, deg, j);
        if (DET) mark_dependants(a, vj, lj, hj, lane, 32);
        else
            for (int64_t e = lj + lane; e < hj; e += 32) a.flag_cur[__ldg(&a.tgt[e])] = 1;
    }
}

// MG over one row.  CHUNKED: the R_H chunks of _chunk_bounds (lpa.py:110-118)
// are cut by arc position while the row streams; each finished chunk is
// folded into parts[0] right away -- the same replay sequence as
// sk = parts[0]; sk.merge(parts[1]); ... (lpa.py:179-186, sketch.py:76-91).
template <int K, bool CHUNKED, class V>
struct MgLane {
    static constexpr bool kHasRescan = true;
    MgSketchDev<K, V> S, part;
    int k, p;
    int64_t base, rem, next;
    __device__ __forceinline__ void init(int k_, int32_t, int64_t deg, int P) {
        k = K > 0 ? K : k_;
        S.reset(k);
        if (CHUNKED) {
            part.reset(k);
            p = 0;
            base = deg / P;
            rem = deg % P;
            next = base + (rem > 0 ? 1 : 0);
        }
    }
    __device__ __forceinline__ void end_chunk() {
        if (p == 0) {
            S = part;
        } else {
#pragma unroll
            for (int i = 0; i < KArr<K>::v; ++i) {
                if (K == 0 && i >= k) break;
                if (part.val[i] > (V)0) S.acc(part.key[i], part.val[i], k);
            }
        }
        part.reset(k);
        ++p;
        next += base + (p < rem ? 1 : 0);
    }
    template <class W>
    __device__ __forceinline__ void on(int64_t pos, bool valid, int32_t c, W w) {
        if (CHUNKED) {
            if (pos == next) end_chunk();
            if (valid) part.acc(c, (V)w, k);
        } else if (valid) {
            S.acc(c, (V)w, k);
        }
    }
    __device__ __forceinline__ void finish() {
        if (CHUNKED) end_chunk();
    }
    __device__ __forceinline__ void rescan_begin() { S.clear_values(k); }
    template <class W>
    __device__ __forceinline__ void rescan(int32_t c, W w) { S.rescan_add(c, (V)w, k); }
    __device__ __forceinline__ int32_t result(int32_t cur) const {
        int32_t b;
        return S.max_key(k, b) ? b : cur;  // lpa.py:192-193
    }
};

// BM over one row: one BmState(cur, 0) per chunk, reduce_votes pair-max
// (lpa.py:137-150); unchunked rows are a single vote.
template <bool CHUNKED, class V>
struct BmLane {
    static constexpr bool kHasRescan = false;
    BmVote<V> st, best;
    int32_t cur0;
    int p;
    int64_t base, rem, next;
    __device__ __forceinline__ void init(int, int32_t cur, int64_t deg, int P) {
        cur0 = cur;
        st = BmVote<V>{cur, (V)0};
        if (CHUNKED) {
            p = 0;
            base = deg / P;
            rem = deg % P;
            next = base + (rem > 0 ? 1 : 0);
        }
    }
    __device__ __forceinline__ void end_chunk() {
        if (p == 0 || bm_better(st.w, st.cand, best.w, best.cand)) best = st;
        st = BmVote<V>{cur0, (V)0};
        ++p;
        next += base + (p < rem ? 1 : 0);
    }
    template <class W>
    __device__ __forceinline__ void on(int64_t pos, bool valid, int32_t c, W w) {
        if (CHUNKED && pos == next) end_chunk();
        if (valid) st.acc(c, (V)w);
    }
    __device__ __forceinline__ void finish() {
        if (CHUNKED) end_chunk();
        else best = st;
    }
    __device__ __forceinline__ void rescan_begin() {}
    template <class W>
    __device__ __forceinline__ void rescan(int32_t, W) {}
    __device__ __forceinline__ int32_t result(int32_t) const { return best.cand; }
};

template <class W, class Pol, bool DET>
__global__ void __launch_bounds__(kWinThreads) k_lane_win(SweepArgs a, const int32_t *__restrict__ list,
                                                          int64_t count, int round0) {
    constexpr int S = WinS<W>::S;
    __shared__ uint32_t s_lab[kWinWarps][32][S + 1];
    __shared__ W s_w[kWinWarps][32][S + 1];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int32_t v = -1;
    uint8_t f0 = 0;
    bool go = false;
    if (i < count) {
        v = __ldg(&list[i]);
        f0 = a.flag_cur[v];
        go = DET ? (!round0 || f0) : (f0 != 0);
    }
    int64_t lo = 0, deg = 0;
    int32_t cur = 0;
    if (go) {
        if (!DET) a.flag_cur[v] = 0;
        lo = __ldg(&a.off[v]);
        deg = __ldg(&a.off[v + 1]) - lo;
        cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
    }
    Pol pol;
    pol.init(a.k, cur, deg, a.parts);
    bool lower_changed = false;
    window_streams<W, DET, false>(a, s_lab[wib], s_w[wib], lane, lo, deg, v, lower_changed,
                                  [&](int64_t pos, bool valid, int32_t c, W w) { pol.on(pos, valid, c, w); });
    if (go && deg) pol.finish();
    if (Pol::kHasRescan && a.scan_double) {
        pol.rescan_begin();
        bool dummy = false;
        window_streams<W, DET, false>(a, s_lab[wib], s_w[wib], lane, lo, deg, v, dummy,
                                      [&](int64_t, bool valid, int32_t c, W w) {
                                          if (valid) pol.rescan(c, w);
                                      });
    }
    unsigned long long n_delta = 0;
    const int32_t cand = (go && deg) ? pol.result(cur) : cur;
    const bool T = go && (f0 || (a.symmetric ? lower_changed : lower_in_changed(a, v)));
    lane_finish<DET>(a, go, v, cur, cand, T, lo, deg, n_delta);
    warp_count(a.counters, go ? 1ull : 0ull, (unsigned long long)deg, n_delta);
}

// High degree, MG: warp per vertex, lane g = chunk g of _chunk_bounds(deg,
// R_H) (lpa.py:178-183) with a register sketch, streamed through the window
// tile; then parts[1..] are replayed into parts[0] in order (sketch.py:
// 76-91) on a slot-parallel warp sketch (lane l = slot l).
template <class W, int K, bool DET, class V>
__global__ void __launch_bounds__(kWinThreads) k_mg_hi_win(SweepArgs a, const int32_t *__restrict__ list,
                                                           int64_t count, int round0) {
    constexpr int S = WinS<W>::S;
    __shared__ uint32_t s_lab[kWinWarps][32][S + 1];
    __shared__ W s_w[kWinWarps][32][S + 1];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= count) return;  // warp-uniform
    if (((a.dbg & 4) && wid != 0) || ((a.dbg & 8) && wid == 0)) return;  // timing experiments only
    const int32_t v = __ldg(&list[wid]);
    const uint8_t f0 = a.flag_cur[v];
    if (DET) {
        if (round0 && !f0) return;
    } else {
        if (!f0) return;
        __syncwarp();
        if (lane == 0) a.flag_cur[v] = 0;
    }
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int64_t deg = hi - lo;
    const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
    const int k = K > 0 ? K : a.k;
    const int P = a.parts;
    bool lower_changed = false;
    WarpSketch<V> S_{0, (V)0};
    for (int b0 = 0; b0 < P; b0 += 32) {
        const int p = b0 + lane;
        MgSketchDev<K, V> part;
        part.reset(k);
        int64_t cs = 0, ce = 0;
        if (p < P) chunk_bounds(deg, P, p, cs, ce);
        window_streams<W, DET, true>(a, s_lab[wib], s_w[wib], lane, lo + cs, ce - cs, v, lower_changed,
                               [&](int64_t, bool valid, int32_t c, double w) {
                                         if (valid && !(a.dbg & 2)) part.acc(c, w, k);
                                     });
        int first = 0;
        if (b0 == 0) {  // sk = parts[0]
#pragma unroll
            for (int i = 0; i < KArr<K>::v; ++i) {
                if (K == 0 && i >= k) break;
                int32_t kk = __shfl_sync(0xffffffffu, part.key[i], 0);
                V vv = __shfl_sync(0xffffffffu, part.val[i], 0);
                if (lane == i) { S_.key = kk; S_.val = vv; }
            }
            first = 1;
        }
        const int nb = min(32, P - b0);
        unsigned nz = 0;
#pragma unroll
        for (int i = 0; i < KArr<K>::v; ++i) {
            if (K == 0 && i >= k) break;
            if (part.val[i] > (V)0) nz |= 1u << (i & 31);
        }
        for (int q = first; q < nb; ++q) {
            const unsigned mq = __shfl_sync(0xffffffffu, nz, q);
            if (!mq) continue;
#pragma unroll
            for (int i = 0; i < KArr<K>::v; ++i) {
                if (K == 0 && i >= k) break;
                if (!(mq & (1u << (i & 31)))) continue;
                int32_t c = __shfl_sync(0xffffffffu, part.key[i], q);
                V w = __shfl_sync(0xffffffffu, part.val[i], q);
                if (!(a.dbg & 1)) S_.acc(lane, k, c, w);
            }
        }
    }
    if (a.scan_double) {  // exact per-key re-count in adjacency order
        S_.val = (V)0;
        bool dummy = false;
        for (int64_t base = lo; base < hi; base += 32) {
            int64_t x = base + lane;
            int32_t c = 0;
            V w = (V)0;
            bool ok = false;
            if (x < hi) {
                int32_t t = __ldg(&a.tgt[x]);
                if (t != v) {
                    ok = true;
                    c = DET ? det_label(a, t, v, dummy) : async_label(a, t);
                    w = (V)arc_weight<W>(a, x);
                }
            }
            unsigned okm = __ballot_sync(0xffffffffu, ok);
            while (okm) {
                int j = __ffs(okm) - 1;
                okm &= okm - 1;
                int32_t cj = __shfl_sync(0xffffffffu, c, j);
                V wj = __shfl_sync(0xffffffffu, w, j);
                S_.rescan_add(lane, k, cj, wj);
            }
        }
    }
    int32_t best;
    const bool found = S_.max_key(lane, k, best);
    warp_hi_finish<DET>(a, v, cur, found ? best : cur, f0, lower_changed, lo, hi, lane);
}

// High degree, BM: one vote per chunk, pair-max reduce (lpa.py:143-150).
template <class W, bool DET, class V>
__global__ void __launch_bounds__(kWinThreads) k_bm_hi_win(SweepArgs a, const int32_t *__restrict__ list,
                                                           int64_t count, int round0) {
    constexpr int S = WinS<W>::S;
    __shared__ uint32_t s_lab[kWinWarps][32][S + 1];
    __shared__ W s_w[kWinWarps][32][S + 1];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= count) return;
    const int32_t v = __ldg(&list[wid]);
    const uint8_t f0 = a.flag_cur[v];
    if (DET) {
        if (round0 && !f0) return;
    } else {
        if (!f0) return;
        __syncwarp();
        if (lane == 0) a.flag_cur[v] = 0;
    }
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int64_t deg = hi - lo;
    const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
    const int P = a.parts;
    bool lower_changed = false;
    bool have = false;
    int32_t bc = 0;
    V bw = (V)0;
    for (int b0 = 0; b0 < P; b0 += 32) {
        const int p = b0 + lane;
        int64_t cs = 0, ce = 0;
        if (p < P) chunk_bounds(deg, P, p, cs, ce);
        BmVote<V> st{cur, (V)0};
        window_streams<W, DET, true>(a, s_lab[wib], s_w[wib], lane, lo + cs, ce - cs, v, lower_changed,
                               [&](int64_t, bool valid, int32_t c, double w) {
                                         if (valid) st.acc(c, w);
                                     });
        if (p < P && (!have || bm_better(st.w, st.cand, bw, bc))) { bc = st.cand; bw = st.w; have = true; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        int oh = __shfl_xor_sync(0xffffffffu, (int)have, o);
        int32_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
        V ow = __shfl_xor_sync(0xffffffffu, bw, o);
        if (oh && (!have || bm_better(ow, oc, bw, bc))) { bc = oc; bw = ow; have = true; }
    }
    warp_hi_finish<DET>(a, v, cur, bc, f0, lower_changed, lo, hi, lane);
}

// ================================================================== giant vertices
// deg >= giant threshold: a single warp per vertex would walk deg/32 arcs per
// lane with dependent staging latencies on every window -- the tail of every
// heavy phase (8 ms for the 406k-degree hub at RMAT s24).  Two kernels:
//  (A) gather: a block per giant materialises its arcs' (label word, weight)
//      stream -- lower neighbours' L1|changed, higher neighbours' L0, self
//      arcs weight 0 -- coalesced and fully parallel;
//  (B) scan: a warp per giant, lane g replays chunk g from that contiguous
//      buffer with register double-buffered prefetch, so the per-lane chain
//      runs at ALU speed; then the ordered merge as in k_mg_hi_win.
constexpr int kGatherThreads = 256;

template <class W, bool DET>
__global__ void __launch_bounds__(kGatherThreads) k_giant_gather(SweepArgs a, const int32_t *__restrict__ slots,
                                                                 int64_t count, int round0) {
    const int64_t b = blockIdx.x;
    if (b >= count) return;
    const int32_t slot = __ldg(&slots[b]);
    const int32_t v = __ldg(&a.giant_bin[slot]);
    const uint8_t f0 = a.flag_cur[v];
    if (DET ? (round0 && !f0) : !f0) return;
    const W *__restrict__ wts = reinterpret_cast<const W *>(a.w);
    W *gw = reinterpret_cast<W *>(a.gw);
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int64_t base = __ldg(&a.giant_off[slot]) - lo;
    const uint64_t pol = policy_evict_first();
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
        const int32_t t = ld_stream(&a.tgt[e], pol);
        W w = ld_stream(&wts[e], pol);
        uint32_t L = 0;
        if (t == v) {
            w = (W)0;
        } else if (DET) {
            L = __ldcg(&a.lab_new[t]);
            if (t > v && (L >> 31)) L = (uint32_t)__ldg(&a.lab_old[t]);
        } else {
            L = (uint32_t)__ldcg(&a.lab_old[t]);
        }
        a.glab[base + e] = L;
        gw[base + e] = w;
    }
}

// Per-lane replay of [x, end) of a giant's gathered stream, 16-element
// register batches, next batch loaded before the current one is consumed.
template <class W, class F>
__device__ __forceinline__ void giant_stream(const SweepArgs &a, int64_t x, int64_t end, bool &lower_changed, F &&f) {
    constexpr int B = 16;
    const W *gw = reinterpret_cast<const W *>(a.gw);
    uint32_t La[B], Lb[B];
    W wa[B], wb[B];
    auto load = [&](uint32_t (&L)[B], W (&w)[B], int64_t p) {
#pragma unroll
        for (int j = 0; j < B; ++j) {
            if (p + j < end) {
                L[j] = __ldcg(&a.glab[p + j]);
                w[j] = __ldcg(&gw[p + j]);
            } else {
                L[j] = 0;
                w[j] = (W)0;
            }
        }
    };
    auto use = [&](const uint32_t (&L)[B], const W (&w)[B]) {
#pragma unroll
        for (int j = 0; j < B; ++j) {
            if (w[j] != (W)0) {
                lower_changed |= (L[j] >> 31) != 0;
                f((int32_t)(L[j] & SLPA_LMASK), w[j]);
            }
        }
    };
    if (x >= end) return;
    load(La, wa, x);
    for (;;) {
        const int64_t nx = x + B;
        if (nx < end) load(Lb, wb, nx);
        use(La, wa);
        if (nx >= end) break;
        x = nx + B;
        if (x < end) load(La, wa, x);
        use(Lb, wb);
        if (x >= end) break;
    }
}

template <class W, int K, bool DET, class V>
__global__ void __launch_bounds__(kWinThreads) k_mg_giant(SweepArgs a, const int32_t *__restrict__ slots,
                                                          int64_t count, int round0) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= count) return;
    const int32_t slot = __ldg(&slots[wid]);
    const int32_t v = __ldg(&a.giant_bin[slot]);
    const uint8_t f0 = a.flag_cur[v];
    if (DET) {
        if (round0 && !f0) return;
    } else {
        if (!f0) return;
        __syncwarp();
        if (lane == 0) a.flag_cur[v] = 0;
    }
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int64_t deg = hi - lo;
    const int64_t base = __ldg(&a.giant_off[slot]);
    const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
    const int k = K > 0 ? K : a.k;
    const int P = a.parts;
    bool lower_changed = false;
    WarpSketch<V> S_{0, (V)0};
    for (int b0 = 0; b0 < P; b0 += 32) {
        const int p = b0 + lane;
        MgSketchDev<K, V> part;
        part.reset(k);
        int64_t cs = 0, ce = 0;
        if (p < P) chunk_bounds(deg, P, p, cs, ce);
        giant_stream<W>(a, base + cs, base + ce, lower_changed, [&](int32_t c, W w) { part.acc(c, (V)w, k); });
        int first = 0;
        if (b0 == 0) {
#pragma unroll
            for (int i = 0; i < KArr<K>::v; ++i) {
                if (K == 0 && i >= k) break;
                int32_t kk = __shfl_sync(0xffffffffu, part.key[i], 0);
                V vv = __shfl_sync(0xffffffffu, part.val[i], 0);
                if (lane == i) { S_.key = kk; S_.val = vv; }
            }
            first = 1;
        }
        const int nb = min(32, P - b0);
        unsigned nz = 0;
#pragma unroll
        for (int i = 0; i < KArr<K>::v; ++i) {
            if (K == 0 && i >= k) break;
            if (part.val[i] > (V)0) nz |= 1u << (i & 31);
        }
        for (int q = first; q < nb; ++q) {
            const unsigned mq = __shfl_sync(0xffffffffu, nz, q);
            if (!mq) continue;
#pragma unroll
            for (int i = 0; i < KArr<K>::v; ++i) {
                if (K == 0 && i >= k) break;
                if (!(mq & (1u << (i & 31)))) continue;
                int32_t c = __shfl_sync(0xffffffffu, part.key[i], q);
                V w = __shfl_sync(0xffffffffu, part.val[i], q);
                S_.acc(lane, k, c, w);
            }
        }
    }
    if (a.scan_double) {  // exact per-key re-count in adjacency order, from the gathered stream
        S_.val = (V)0;
        const W *gw = reinterpret_cast<const W *>(a.gw);
        for (int64_t b = 0; b < deg; b += 32) {
            const int64_t x = b + lane;
            int32_t c = 0;
            V w = (V)0;
            if (x < deg) {
                w = (V)__ldcg(&gw[base + x]);
                c = (int32_t)(__ldcg(&a.glab[base + x]) & SLPA_LMASK);
            }
            unsigned okm = __ballot_sync(0xffffffffu, w != (V)0);
            while (okm) {
                int j = __ffs(okm) - 1;
                okm &= okm - 1;
                S_.rescan_add(lane, k, __shfl_sync(0xffffffffu, c, j), __shfl_sync(0xffffffffu, w, j));
            }
        }
    }
    int32_t best;
    const bool found = S_.max_key(lane, k, best);
    warp_hi_finish<DET>(a, v, cur, found ? best : cur, f0, lower_changed, lo, hi, lane);
}

template <class W, bool DET, class V>
__global__ void __launch_bounds__(kWinThreads) k_bm_giant(SweepArgs a, const int32_t *__restrict__ slots,
                                                          int64_t count, int round0) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= count) return;
    const int32_t slot = __ldg(&slots[wid]);
    const int32_t v = __ldg(&a.giant_bin[slot]);
    const uint8_t f0 = a.flag_cur[v];
    if (DET) {
        if (round0 && !f0) return;
    } else {
        if (!f0) return;
        __syncwarp();
        if (lane == 0) a.flag_cur[v] = 0;
    }
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int64_t deg = hi - lo;
    const int64_t base = __ldg(&a.giant_off[slot]);
    const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
    const int P = a.parts;
    bool lower_changed = false, have = false;
    int32_t bc = 0;
    V bw = (V)0;
    for (int p = lane; p < P; p += 32) {
        int64_t cs, ce;
        chunk_bounds(deg, P, p, cs, ce);
        BmVote<V> st{cur, (V)0};
        giant_stream<W>(a, base + cs, base + ce, lower_changed, [&](int32_t c, W w) { st.acc(c, (V)w); });
        if (!have || bm_better(st.w, st.cand, bw, bc)) { bc = st.cand; bw = st.w; have = true; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        int oh = __shfl_xor_sync(0xffffffffu, (int)have, o);
        int32_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
        V ow = __shfl_xor_sync(0xffffffffu, bw, o);
        if (oh && (!have || bm_better(ow, oc, bw, bc))) { bc = oc; bw = ow; have = true; }
    }
    warp_hi_finish<DET>(a, v, cur, bc, f0, lower_changed, lo, hi, lane);
}

// ================================================================== exact
// select_label_exact (lpa.py:92-107): per-label totals summed in adjacency
// order (np.bincount order), argmax = smallest label among ties.  One thread
// per vertex, O(deg^2) -- the correctness path for the quality baseline.
template <class W, bool DET>
__global__ void __launch_bounds__(kThreads) k_exact(SweepArgs a, const int32_t *__restrict__ list, int64_t count,
                                                    int round0) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long n_eval = 0, n_arcs = 0, n_delta = 0;
    int32_t v = 0;
    uint8_t f0 = 0;
    bool go = false;
    if (i < count) {
        v = __ldg(&list[i]);
        f0 = a.flag_cur[v];
        go = DET ? (!round0 || f0) : (f0 != 0);
    }
    if (go) {
        if (!DET) a.flag_cur[v] = 0;
        const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
        const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
        bool lower_changed = false, dummy = false;
        bool found = false;
        int32_t best = 0;
        double bw = 0.0;
        for (int64_t e1 = lo; e1 < hi; ++e1) {
            int32_t t1 = __ldg(&a.tgt[e1]);
            if (t1 == v) continue;
            int32_t c1 = DET ? det_label(a, t1, v, lower_changed) : async_label(a, t1);
            bool seen = false;
            for (int64_t e0 = lo; e0 < e1 && !seen; ++e0) {
                int32_t t0 = __ldg(&a.tgt[e0]);
                if (t0 == v) continue;
                int32_t c0 = DET ? det_label(a, t0, v, dummy) : async_label(a, t0);
                seen = (c0 == c1);
            }
            if (seen) continue;
            double tot = 0.0;
            for (int64_t e2 = e1; e2 < hi; ++e2) {
                int32_t t2 = __ldg(&a.tgt[e2]);
                if (t2 == v) continue;
                int32_t c2 = DET ? det_label(a, t2, v, dummy) : async_label(a, t2);
                if (c2 == c1) tot += arc_weight<W>(a, e2);
            }
            if (!found || tot > bw || (tot == bw && c1 < best)) { best = c1; bw = tot; found = true; }
        }
        const int32_t cand = found ? best : cur;
        n_eval = 1;
        n_arcs = (unsigned long long)(hi - lo);
        if (DET) {
            bool T = f0 || (a.symmetric ? lower_changed : lower_in_changed(a, v));
            det_commit_output(a, v, cur, cand, T, lo, hi);
        } else {
            async_commit_output(a, v, cur, cand, lo, hi, n_delta);
        }
    }
    warp_count(a.counters, n_eval, n_arcs, n_delta);
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
            for (int64_t e = lo; e < hi; ++e) {
                int32_t t = __ldg(&a.tgt[e]);
                if (t <= v) a.flag_next[t] = 1;
            }
        }
    }
    warp_count(a.counters, 0, 0, d);
}

__global__ void __launch_bounds__(kThreads) k_commit_hi(SweepArgs a, const int32_t *__restrict__ list, int64_t count) {
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= count) return;
    const int32_t v = __ldg(&list[wid]);
    uint32_t wv = a.lab_new[v];
    if (!(wv & SLPA_CHG)) return;
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    for (int64_t e = lo + lane; e < hi; e += 32) {
        int32_t t = __ldg(&a.tgt[e]);
        if (t <= v) a.flag_next[t] = 1;
    }
    __syncwarp();
    if (lane == 0) {
        int32_t c = (int32_t)(wv & SLPA_LMASK);
        a.lab_old[v] = c;
        a.lab_new[v] = (uint32_t)c;
        ctr_add(a.counters, CNT_DELTA, 1ull);
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
typedef void (*EvalKernel)(SweepArgs, const int32_t *, int64_t, int);

// lo: one lane per vertex, one sketch; mid: one lane per vertex, R_H chunks;
// hi: one warp per vertex, lane = chunk (or thread-per-vertex for `exact`);
// giant: gather + warp-per-vertex replay.
struct KernelSet {
    EvalKernel lo, mid, hi, gather, giant;
    int lo_threads, hi_threads;
    bool hi_is_warp;
};

template <class W, bool DET, class V>
KernelSet pick_kernels(const slpa_config *cfg) {
    if (cfg->variant == SLPA_VARIANT_EXACT)
        return {k_exact<W, DET>, k_exact<W, DET>, k_exact<W, DET>, nullptr, nullptr, kThreads, kThreads, false};
    if (cfg->variant == SLPA_VARIANT_BM)
        return {k_lane_win<W, BmLane<false, V>, DET>, k_lane_win<W, BmLane<true, V>, DET>, k_bm_hi_win<W, DET, V>,
                k_giant_gather<W, DET>, k_bm_giant<W, DET, V>, kWinThreads, kWinThreads, true};
    if (cfg->sketch_slots == 8)
        return {k_lane_win<W, MgLane<8, false, V>, DET>, k_lane_win<W, MgLane<8, true, V>, DET>,
                k_mg_hi_win<W, 8, DET, V>, k_giant_gather<W, DET>, k_mg_giant<W, 8, DET, V>, kWinThreads,
                kWinThreads, true};
    return {k_lane_win<W, MgLane<0, false, V>, DET>, k_lane_win<W, MgLane<0, true, V>, DET>,
            k_mg_hi_win<W, 0, DET, V>, k_giant_gather<W, DET>, k_mg_giant<W, 0, DET, V>, kWinThreads, kWinThreads,
            true};
}

// Integer sketch values when the exactness precondition holds (slpa_sketch.cuh).
KernelSet kernels_for(const slpa_ctx *ctx, const slpa_config *cfg, bool det) {
    static const int force_fp64 = [] {
        const char *e = getenv("SLPA_FORCE_FP64");
        return e ? atoi(e) : 0;
    }();
    const bool iv = ctx->g.int_weights && !force_fp64;
    if (ctx->g.w_f64) {
        if (iv) return det ? pick_kernels<double, true, uint32_t>(cfg) : pick_kernels<double, false, uint32_t>(cfg);
        return det ? pick_kernels<double, true, double>(cfg) : pick_kernels<double, false, double>(cfg);
    }
    if (iv) return det ? pick_kernels<float, true, uint32_t>(cfg) : pick_kernels<float, false, uint32_t>(cfg);
    return det ? pick_kernels<float, true, double>(cfg) : pick_kernels<float, false, double>(cfg);
}

SweepArgs make_args(slpa_ctx *ctx, const slpa_config *cfg, int pickless) {
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
    static const int dbg = [] {
        const char *e = getenv("SLPA_DEBUG_SKIP");
        return e ? atoi(e) : 0;
    }();
    a.dbg = dbg;
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
void timed_launch(slpa_ctx *ctx, int cls, int nlaunch, F &&fn) {
    ctx->stats.kernel_launches += nlaunch;
    if (!ctx->prof_on) {
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
}

void launch_lane(slpa_ctx *ctx, EvalKernel k, int threads, const SweepArgs &a, const int32_t *list, int64_t cnt,
                 int round0, int cls) {
    if (cnt <= 0) return;
    timed_launch(ctx, cls, 1, [&] {
        k<<<grid_for(cnt, threads), threads, 0, ctx->stream>>>(a, list, cnt, round0);
        CUDA_TRY(cudaGetLastError());
    });
}

void launch_hi(slpa_ctx *ctx, const KernelSet &ks, const SweepArgs &a, const int32_t *list, int64_t cnt, int round0,
               int cls) {
    if (cnt <= 0) return;
    timed_launch(ctx, cls, 1, [&] {
        const int64_t items = ks.hi_is_warp ? cnt * 32 : cnt;
        ks.hi<<<grid_for(items, ks.hi_threads), ks.hi_threads, 0, ctx->stream>>>(a, list, cnt, round0);
        CUDA_TRY(cudaGetLastError());
    });
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
        ks.gather<<<(unsigned)cnt, kGatherThreads, 0, gs>>>(a, slots, cnt, round0);
        ks.giant<<<grid_for(cnt * 32, kWinThreads), kWinThreads, 0, gs>>>(a, slots, cnt, round0);
        CUDA_TRY(cudaGetLastError());
    });
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

__global__ void k_iota(int32_t *out, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)i;
}

}  // namespace

// ====================================================================== drivers
int64_t slpa_sweep_det(slpa_ctx *ctx, const slpa_config *cfg, int pickless) {
    DeviceGraph &g = ctx->g;
    WorkBuffers &wb = ctx->wb;
    cudaStream_t s = ctx->stream;
    const int64_t n = g.n;
    const KernelSet ks = kernels_for(ctx, cfg, true);
    const SweepArgs a = make_args(ctx, cfg, pickless);
    CUDA_TRY(cudaMemsetAsync(wb.counters.p, 0, CNT_TOTAL * sizeof(unsigned long long), s));
    CUDA_TRY(cudaMemsetAsync(wb.flag_b.p, 0, (size_t)n, s));
    for (int c = 0; c < CNT_N; ++c) ctx->h_sum[c] = 0;
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
        launch_lane(ctx, ks.mid, ks.lo_threads, a, g.bin_mid.p, g.n_mid, 1, SLPA_PROF_EVAL_MID0);
    }
    launch_lane(ctx, ks.lo, ks.lo_threads, a, g.bin_lo.p, g.n_lo, 1, SLPA_PROF_EVAL_LO0);
    int64_t rounds = 1;
    unsigned long long evals0 = 0, arcs0 = 0;
    bool first = true;
    unsigned long long *cur_lo = wb.counters.p + CNT_LO * CNT_STRIPES, *cur_mid = wb.counters.p + CNT_MID * CNT_STRIPES,
                       *cur_hi = wb.counters.p + CNT_HI * CNT_STRIPES,
                       *cur_giant = wb.counters.p + CNT_GIANT * CNT_STRIPES;
    bool pend_any = defer != 0;
    for (;;) {
        giant_join(ctx);
        CUDA_TRY(cudaMemsetAsync(cur_lo, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(cur_mid, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(cur_hi, 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaMemsetAsync(cur_giant, 0, sizeof(unsigned long long), s));
        timed_launch(ctx, SLPA_PROF_COMPACT, 4, [&] {
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
        CUDA_TRY(cudaMemsetAsync(wb.dirty_a.p, 0, (size_t)nwords * sizeof(uint32_t), s));
        read_counters(ctx);
        if (first) {
            evals0 = ctx->h_sum[CNT_EVALS] + ctx->h_sum[CNT_EVALS_HI];
            arcs0 = ctx->h_sum[CNT_ARCS] + ctx->h_sum[CNT_ARCS_HI];
            first = false;
        }
        int64_t nlo = (int64_t)ctx->h_sum[CNT_LO], nmid = (int64_t)ctx->h_sum[CNT_MID],
                nhi = (int64_t)ctx->h_sum[CNT_HI], ngiant = (int64_t)ctx->h_sum[CNT_GIANT];
        if (defer && nlo == 0 && pend_any) {  // light vertices quiet: run the pending heavy ones
            timed_launch(ctx, SLPA_PROF_COMPACT, 3, [&] {
                launch_filter(s, g.bin_hi.p, g.n_hi, wb.dirty_b.p, wb.wl_hi.p, cur_hi);
                launch_filter(s, g.bin_mid.p, g.n_mid, wb.dirty_b.p, wb.wl_mid.p, cur_mid);
                launch_filter(s, g.bin_giant.p, g.n_giant, wb.dirty_b.p, wb.wl_giant.p, cur_giant, 1);
                CUDA_TRY(cudaGetLastError());
            });
            CUDA_TRY(cudaMemsetAsync(wb.dirty_b.p, 0, (size_t)nwords * sizeof(uint32_t), s));
            read_counters(ctx);
            nmid = (int64_t)ctx->h_sum[CNT_MID];
            nhi = (int64_t)ctx->h_sum[CNT_HI];
            ngiant = (int64_t)ctx->h_sum[CNT_GIANT];
        }
        if (nlo == 0 && nmid == 0 && nhi == 0 && ngiant == 0) break;
        pend_any = defer != 0;
        launch_giant(ctx, ks, a, wb.wl_giant.p, ngiant, 0);
        launch_hi(ctx, ks, a, wb.wl_hi.p, nhi, 0, SLPA_PROF_EVAL_HIK);
        launch_lane(ctx, ks.lo, ks.lo_threads, a, wb.wl_lo.p, nlo, 0, SLPA_PROF_EVAL_LOK);
        launch_lane(ctx, ks.mid, ks.lo_threads, a, wb.wl_mid.p, nmid, 0, SLPA_PROF_EVAL_MIDK);
        ++rounds;
    }
    giant_join(ctx);
    const unsigned long long evals = ctx->h_sum[CNT_EVALS] + ctx->h_sum[CNT_EVALS_HI];
    const unsigned long long arcs = ctx->h_sum[CNT_ARCS] + ctx->h_sum[CNT_ARCS_HI];
    // commit: L0 <- L1, delta, next-sweep flags
    timed_launch(ctx, SLPA_PROF_COMMIT, 4, [&] {
        if (g.n_lo > 0) k_commit_lo<<<grid_for(g.n_lo, kThreads), kThreads, 0, s>>>(a, g.bin_lo.p, g.n_lo);
        if (g.n_mid > 0) k_commit_hi<<<grid_for(g.n_mid * 32, kThreads), kThreads, 0, s>>>(a, g.bin_mid.p, g.n_mid);
        if (g.n_hi > 0) k_commit_hi<<<grid_for(g.n_hi * 32, kThreads), kThreads, 0, s>>>(a, g.bin_hi.p, g.n_hi);
        if (g.n_giant > 0)
            k_commit_hi<<<grid_for(g.n_giant * 32, kThreads), kThreads, 0, s>>>(a, g.bin_giant.p, g.n_giant);
        CUDA_TRY(cudaGetLastError());
    });
    read_counters(ctx);
    std::swap(wb.flag_a, wb.flag_b);
    ctx->stats.rounds += rounds;
    ctx->stats.vertex_evals += (int64_t)evals;
    ctx->stats.arc_reads += (int64_t)arcs;
    ctx->stats.first_evals += (int64_t)evals0;
    ctx->stats.first_arcs += (int64_t)arcs0;
    return (int64_t)ctx->h_sum[CNT_DELTA];
}

int64_t slpa_sweep_async(slpa_ctx *ctx, const slpa_config *cfg, int pickless) {
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
    launch_lane(ctx, ks.mid, ks.lo_threads, a, g.bin_mid.p, g.n_mid, 1, SLPA_PROF_EVAL_MID0);
    launch_lane(ctx, ks.lo, ks.lo_threads, a, g.bin_lo.p, g.n_lo, 1, SLPA_PROF_EVAL_LO0);
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
    ctx->stats.rounds += 1;
    ctx->stats.vertex_evals += ev;
    ctx->stats.arc_reads += ar;
    ctx->stats.first_evals += ev;
    ctx->stats.first_arcs += ar;
    return (int64_t)ctx->h_sum[CNT_DELTA];
}

void slpa_init_labels(slpa_ctx *ctx) {
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
    if (ctx->g.has_order) {
        k_pos_to_id_i32<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(src, ctx->wb.io_labels.p, ctx->g.ids.p, n);
        CUDA_TRY(cudaGetLastError());
        src = ctx->wb.io_labels.p;
    }
    CUDA_TRY(cudaMemcpyAsync(host, src, n * sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
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
