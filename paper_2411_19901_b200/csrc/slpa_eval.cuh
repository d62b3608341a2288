// slpa_eval.cuh -- the vertex-evaluation kernels of a sweep (templates only;
// instantiated per weight type / sketch value type / mode in slpa_eval_*.cu so
// the heavy template code compiles in parallel translation units).
#pragma once
#include <cstdlib>
#include "slpa_sketch.cuh"
#include "slpa_internal.cuh"

// minimum resident blocks per SM for the two bulk kernels (register caps; A/B builds)
#ifndef SLPA_MERGE_MINB
#define SLPA_MERGE_MINB 1
#endif
#ifndef SLPA_HI_THREADS
#define SLPA_HI_THREADS 256
#endif
#ifndef SLPA_HI_MINB
#define SLPA_HI_MINB 1
#endif
// light rows: 3 blocks of 256 threads per SM (85-register cap, a 24-byte
// spill outside the batch loop): k-mer 151 -> 142 ms, grid 14.8 -> 12.8 ms per run
#ifndef SLPA_LO_MINB
#define SLPA_LO_MINB 3
#endif


namespace {

constexpr int kThreads = 256;
#ifndef SLPA_GCS_DEPTH
#define SLPA_GCS_DEPTH 8
#endif
#ifndef SLPA_GIANT_RING
#define SLPA_GIANT_RING 4
#endif
constexpr int kGiantWarps = 8;  // block-per-vertex kernels: 8 warps x 4 groups = 32 chunks

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

// One gather per arc (streaming kernels): a lower neighbour's word from
// lab_new (L1 | changed bit, written this sweep -> L2 load), a higher one's
// L0 straight from lab_old (read-only during the rounds, no changed bit), so
// no dependent second load; async mode reads the in-place labels.
template <bool DET>
__device__ __forceinline__ uint32_t gather_word(const SweepArgs &a, int32_t t, int32_t v) {
    if (!DET) return (uint32_t)__ldcg(&a.lab_old[t]);
    return t < v ? __ldcg(&a.lab_new[t]) : (uint32_t)__ldg(&a.lab_old[t]);
}

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

// Profiling: record whether v's evaluation took its turn (T).  The last
// evaluation of a sweep is the fixpoint's, so at the end of the sweep the
// bitmap is exactly the set of vertices the sequential sweep processes
// (lpa.py:212-216); vertices never evaluated have T = 0.
__device__ __forceinline__ void record_turn(const SweepArgs &a, int32_t v, bool T) {
    if (!a.tbits) return;
    const uint32_t bit = 1u << (v & 31);
    if (T) atomicOr(&a.tbits[v >> 5], bit);
    else atomicAnd(&a.tbits[v >> 5], ~bit);
}

// Finish one deterministic evaluation (thread-per-vertex flavour).
__device__ __forceinline__ void det_commit_output(const SweepArgs &a, int32_t v, int32_t cur, int32_t cand, bool T,
                                                  int64_t lo, int64_t hi) {
    bool chg = T && cand != cur && (!a.pickless || cand < cur);
    record_turn(a, v, T);
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
        if (lane == 0) record_turn(a, v, T);
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

// Warp-per-giant kernels (k_mg_giant, k_bm_giant) run 4-warp blocks.
constexpr int kWinWarps = 4;
constexpr int kWinThreads = kWinWarps * 32;

// ================================================================== direct streaming
// Every lane streams its own arc range [start, start + len) in 32-byte aligned
// batches of 8 arcs: one 256-bit load of targets, one (float) or two (double)
// 256-bit loads of weights, the batch's 8 label gathers issued together, and
// the next batch's targets / weights requested before the current batch is
// consumed.  No shared memory and no warp collectives, so lanes of one warp
// may stream ranges of different lengths.  Arcs of the batch outside the range
// are masked (the buffers carry tail padding, slpa_internal.cuh); self arcs
// are passed to `consume` as invalid so chunk positions stay exact.
constexpr int kBatch = 8;

__device__ __forceinline__ void ld8(const int32_t *p, int32_t (&r)[8], uint64_t pol) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld8(const uint32_t *p, uint32_t (&r)[8]) {  // scratch read once: streaming
    asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld8(const float *p, float (&r)[8], uint64_t pol) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld8(const double *p, double (&r)[8], uint64_t pol) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
                 : "l"(p), "l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=d"(r[4]), "=d"(r[5]), "=d"(r[6]), "=d"(r[7])
                 : "l"(p + 4), "l"(pol));
}
__device__ __forceinline__ void ld8_cg(const float *p, float (&r)[8]) {
    asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld8_cg(const double *p, double (&r)[8]) {
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[4]), "=d"(r[5]), "=d"(r[6]), "=d"(r[7]) : "l"(p + 4));
}

// Unaligned flavour for short ranges (the chunks of a high-degree row): the
// batches start at `start`, so only the last one is partial; targets and
// weights are scalar loads that stay in L1 for the lane's next batch.
template <class W, bool DET, class Consume>
__device__ __forceinline__ void lane_stream_u(const SweepArgs &a, int64_t start, int64_t len, int32_t v,
                                              bool &lower_changed, Consume &&consume) {
    if (len <= 0) return;
    const W *__restrict__ wts = reinterpret_cast<const W *>(a.w);
    int32_t t[kBatch];
    W w[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
        const bool in = j < len;
        t[j] = in ? __ldg(&a.tgt[start + j]) : v;
        w[j] = in ? __ldg(&wts[start + j]) : (W)0;
    }
    for (int64_t x0 = 0;;) {
        uint32_t L[kBatch];
        if (DET && a.ident) {  // round 0 of the first sweep: a neighbour's label is its id (one branch per batch)
#pragma unroll
            for (int j = 0; j < kBatch; ++j) L[j] = t[j] != v ? (uint32_t)t[j] : 0u;
        } else {
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                L[j] = 0;
                if (t[j] != v) L[j] = gather_word<DET>(a, t[j], v);
            }
        }
        const int64_t nx = x0 + kBatch;
        int32_t tn[kBatch];
        W wn[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {  // next batch requested before this one is consumed
            const bool in = nx + j < len;
            tn[j] = in ? __ldg(&a.tgt[start + nx + j]) : v;
            wn[j] = in ? __ldg(&wts[start + nx + j]) : (W)0;
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            if (x0 + j < len) {
                const bool valid = t[j] != v;
                if (DET) lower_changed |= valid && (L[j] >> 31) != 0;
                consume(x0 + j, valid, (int32_t)(L[j] & SLPA_LMASK), w[j]);
            }
        }
        if (nx >= len) break;
        x0 = nx;
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            t[j] = tn[j];
            w[j] = wn[j];
        }
    }
}

// Three-stage flavour for long ranges: while batch i is consumed, the label
// gathers of batch i+1 and the target / weight loads of batch i+2 are in
// flight, so a long chunk streams at the speed of its sketch chain.
template <class W, bool DET>
__device__ __forceinline__ void ld_batch_u(const SweepArgs &a, const W *__restrict__ wts, int64_t start, int64_t x,
                                           int64_t len, int32_t v, int32_t (&t)[kBatch], W (&w)[kBatch]) {
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
        const bool in = x + j < len;
        t[j] = in ? __ldg(&a.tgt[start + x + j]) : v;
        w[j] = in ? __ldg(&wts[start + x + j]) : (W)0;
    }
}

// The high-degree scans gather every word from lab_new, the array L2 keeps
// resident (a higher neighbour's L0 is fetched from lab_old only when its
// changed bit is set): at RMAT s24 reading lab_old directly for every higher
// neighbour doubles the gathers' L2 footprint and measured 13.1 GB of DRAM
// reads per first heavy launch instead of 5.6 GB.
template <bool DET>
__device__ __forceinline__ void gather_batch(const SweepArgs &a, int32_t v, const int32_t (&t)[kBatch],
                                             uint32_t (&L)[kBatch]) {
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
        L[j] = 0;
        if (t[j] != v) L[j] = DET ? __ldcg(&a.lab_new[t[j]]) : (uint32_t)__ldcg(&a.lab_old[t[j]]);
    }
}

template <class W, bool DET, class Consume>
__device__ __forceinline__ void lane_stream_p(const SweepArgs &a, int64_t start, int64_t len, int32_t v,
                                              bool &lower_changed, Consume &&consume) {
    if (len <= 0) return;
    const W *__restrict__ wts = reinterpret_cast<const W *>(a.w);
    int32_t tA[kBatch], tB[kBatch], tC[kBatch];
    W wA[kBatch], wB[kBatch], wC[kBatch];
    uint32_t LA[kBatch], LB[kBatch];
    ld_batch_u<W, DET>(a, wts, start, 0, len, v, tA, wA);
    gather_batch<DET>(a, v, tA, LA);
    ld_batch_u<W, DET>(a, wts, start, kBatch, len, v, tB, wB);
    for (int64_t x0 = 0;;) {
        gather_batch<DET>(a, v, tB, LB);                                // batch i+1 (masked past the end)
        ld_batch_u<W, DET>(a, wts, start, x0 + 2 * kBatch, len, v, tC, wC);  // batch i+2
        if (DET) {  // higher neighbour that changed this sweep: its L0
#pragma unroll
            for (int j = 0; j < kBatch; ++j)
                if (tA[j] > v && (LA[j] >> 31)) LA[j] = (uint32_t)__ldg(&a.lab_old[tA[j]]);
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            if (x0 + j < len) {
                const bool valid = tA[j] != v;
                if (DET) lower_changed |= valid && (LA[j] >> 31) != 0;
                consume(x0 + j, valid, (int32_t)(LA[j] & SLPA_LMASK), wA[j]);
            }
        }
        x0 += kBatch;
        if (x0 >= len) break;
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            tA[j] = tB[j];
            wA[j] = wB[j];
            LA[j] = LB[j];
            tB[j] = tC[j];
            wB[j] = wC[j];
        }
    }
}

// consume(pos, valid, label, w): pos = arc index relative to `start`.
template <class W, bool DET, class Consume>
__device__ __forceinline__ void lane_stream(const SweepArgs &a, int64_t start, int64_t len, int32_t v,
                                            bool &lower_changed, Consume &&consume) {
    if (len <= 0) return;
    const W *__restrict__ wts = reinterpret_cast<const W *>(a.w);
    const uint64_t pol = policy_evict_first();
    const int64_t end = start + len;
    int64_t b = start & ~(int64_t)(kBatch - 1);
    int32_t t[kBatch];
    W w[kBatch];
    ld8(a.tgt + b, t, pol);
    ld8(wts + b, w, pol);
    for (;;) {
        uint32_t L[kBatch];
        unsigned inr = 0, ok = 0;
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const int64_t e = b + j;
            const bool in = e >= start && e < end;
            const bool valid = in && t[j] != v;
            inr |= (unsigned)in << j;
            ok |= (unsigned)valid << j;
        }
        if (DET && a.ident) {  // round 0 of the first sweep: a neighbour's label is its id (one branch per batch)
#pragma unroll
            for (int j = 0; j < kBatch; ++j) L[j] = ((ok >> j) & 1u) ? (uint32_t)t[j] : 0u;
        } else {
#pragma unroll
            for (int j = 0; j < kBatch; ++j) L[j] = ((ok >> j) & 1u) ? gather_word<DET>(a, t[j], v) : 0u;
        }
        const int64_t nb = b + kBatch;
        int32_t tn[kBatch];
        W wn[kBatch];
        const bool more = nb < end;
        if (more) {
            ld8(a.tgt + nb, tn, pol);
            ld8(wts + nb, wn, pol);
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            if ((inr >> j) & 1u) {
                const bool valid = (ok >> j) & 1u;
                if (DET) lower_changed |= valid && (L[j] >> 31) != 0;
                consume(b + j - start, valid, (int32_t)(L[j] & SLPA_LMASK), w[j]);
            }
        }
        if (!more) break;
        b = nb;
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            t[j] = tn[j];
            w[j] = wn[j];
        }
    }
}

// ================================================================== lane kernels
// One lane per vertex.  Lane outputs are written per lane; adjacency walks
// for changed vertices (dependant marks in deterministic mode, neighbour
// flags in async mode) are done by the whole warp, one changed lane at a
// time, so they are coalesced instead of 32 divergent row loops.
template <bool DET, bool LANE_WALK = false>
__device__ __forceinline__ void lane_finish(const SweepArgs &a, bool go, int32_t v, int32_t cur, int32_t cand,
                                            bool T, int64_t lo, int64_t deg, unsigned long long &n_delta) {
    const int lane = threadIdx.x & 31;
    bool walk = false;
    if (go) {
        if (DET) {
            const bool chg = T && cand != cur && (!a.pickless || cand < cur);
            record_turn(a, v, T);
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
    if (LANE_WALK && a.symmetric) {
        // short rows: every changed lane walks its own row, 8 independent
        // target loads in flight per step (a warp-cooperative walk would
        // serialise the changed lanes' rows one round trip each)
        if (walk) {
            const int64_t hi = lo + deg;
            for (int64_t e0 = lo; e0 < hi; e0 += 8) {
                int32_t t[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) t[j] = e0 + j < hi ? __ldg(&a.tgt[e0 + j]) : -1;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (DET) {
                        if (t[j] > v) mark_dirty(a.dirty_next, t[j]);
                    } else if (t[j] >= 0) {
                        a.flag_cur[t[j]] = 1;
                    }
                }
            }
        }
        return;
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
    static constexpr int kMinBlocks = (CHUNKED || K == 0) ? 1 : SLPA_LO_MINB;  // register cap of k_lane_direct
    MgSketchDev<K, V> S, part;
    int k, p;
    int32_t z;
    int64_t base, rem, next;
    __device__ __forceinline__ void init(int k_, int32_t, int64_t deg, int P, int32_t z_) {
        k = K > 0 ? K : k_;
        z = z_;
        S.reset(k, z);
        if (CHUNKED) {
            part.reset(k, z);
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
                const V pv = part.value(i);
                if (pv > (V)0) S.acc(part.key[i], pv, k);
            }
        }
        part.reset(k, z);
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
    static constexpr int kMinBlocks = CHUNKED ? 1 : SLPA_LO_MINB;
    BmVote<V> st, best;
    int32_t cur0;
    int p;
    int64_t base, rem, next;
    __device__ __forceinline__ void init(int, int32_t cur, int64_t deg, int P, int32_t) {
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

// One lane per vertex, every lane streaming its own row directly.
template <class W, class Pol, bool DET>
__global__ void __launch_bounds__(kThreads, Pol::kMinBlocks) k_lane_direct(SweepArgs a, const int32_t *__restrict__ list,
                                                          int64_t count, int round0) {
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
    pol.init(a.k, cur, deg, a.parts, a.zkey);
    bool lower_changed = false;
    // Rows of a warp have similar lengths (degree-ordered bins).  Short rows
    // stream unaligned -- element j of every lane is arc j of its own row, so
    // a warp of degree-d rows runs d accumulate steps; aligned 32-byte
    // batches would scatter those arcs over all 8 batch slots.
    const unsigned maxdeg = __reduce_max_sync(0xffffffffu, (unsigned)deg);
    if (maxdeg <= 8)
        lane_stream_u<W, DET>(a, lo, deg, v, lower_changed,
                              [&](int64_t pos, bool valid, int32_t c, W w) { pol.on(pos, valid, c, w); });
    else
        lane_stream<W, DET>(a, lo, deg, v, lower_changed,
                            [&](int64_t pos, bool valid, int32_t c, W w) { pol.on(pos, valid, c, w); });
    if (go && deg) pol.finish();
    if (Pol::kHasRescan && a.scan_double) {
        pol.rescan_begin();
        bool dummy = false;
        lane_stream<W, DET>(a, lo, deg, v, dummy, [&](int64_t, bool valid, int32_t c, W w) {
            if (valid) pol.rescan(c, w);
        });
    }
    unsigned long long n_delta = 0;
    const int32_t cand = (go && deg) ? pol.result(cur) : cur;
    const bool T = go && (f0 || (a.symmetric ? lower_changed : lower_in_changed(a, v)));
    lane_finish<DET, true>(a, go, v, cur, cand, T, lo, deg, n_delta);
    warp_count(a.counters, go ? 1ull : 0ull, (unsigned long long)deg, n_delta);
}

// Ordered merge of the lanes' part sketches (lane q = parts[b0 + q]) into the
// slot-parallel warp sketch: sk = parts[0]; sk.merge(parts[1]); ...
// (lpa.py:179-186, sketch.py:76-91).
template <int K, class V>
__device__ __forceinline__ void warp_merge_parts(WarpSketch<V> &S_, const MgSketchDev<K, V> &part, int b0, int P,
                                                 int k, int lane) {
    int first = 0;
    if (b0 == 0) {  // sk = parts[0]
#pragma unroll
        for (int i = 0; i < KArr<K>::v; ++i) {
            if (K == 0 && i >= k) break;
            int32_t kk = __shfl_sync(0xffffffffu, part.key[i], 0);
            V vv = __shfl_sync(0xffffffffu, part.value(i), 0);
            if (lane == i) { S_.key = kk; S_.val = vv; }
        }
        first = 1;
    }
    const int nb = min(32, P - b0);
    unsigned nz = 0;
#pragma unroll
    for (int i = 0; i < KArr<K>::v; ++i) {
        if (K == 0 && i >= k) break;
        if (part.value(i) > (V)0) nz |= 1u << (i & 31);
    }
    for (int q = first; q < nb; ++q) {
        const unsigned mq = __shfl_sync(0xffffffffu, nz, q);
        if (!mq) continue;
#pragma unroll
        for (int i = 0; i < KArr<K>::v; ++i) {
            if (K == 0 && i >= k) break;
            if (!(mq & (1u << (i & 31)))) continue;
            int32_t c = __shfl_sync(0xffffffffu, part.key[i], q);
            V w = __shfl_sync(0xffffffffu, part.value(i), q);
            S_.acc(lane, k, c, w);
        }
    }
}

// High degree, MG, direct streaming: warp per vertex, lane g streams chunk g.
template <class W, int K, bool DET, class V>
__global__ void __launch_bounds__(kThreads) k_mg_hi_direct(SweepArgs a, const int32_t *__restrict__ list,
                                                           int64_t count, int round0) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= count) return;  // warp-uniform
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
    WarpSketch<V> S_{a.zkey, (V)0, a.zkey};
    for (int b0 = 0; b0 < P; b0 += 32) {
        const int p = b0 + lane;
        MgSketchDev<K, V> part;
        part.reset(k, a.zkey);
        int64_t cs = 0, ce = 0;
        if (p < P) chunk_bounds(deg, P, p, cs, ce);
        lane_stream_u<W, DET>(a, lo + cs, ce - cs, v, lower_changed, [&](int64_t, bool valid, int32_t c, W w) {
            if (valid) part.acc(c, (V)w, k);
        });
        __syncwarp();
        warp_merge_parts<K, V>(S_, part, b0, P, k, lane);
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
                S_.rescan_add(lane, k, __shfl_sync(0xffffffffu, c, j), __shfl_sync(0xffffffffu, w, j));
            }
        }
    }
    int32_t best;
    const bool found = S_.max_key(lane, k, best);
    warp_hi_finish<DET>(a, v, cur, found ? best : cur, f0, lower_changed, lo, hi, lane);
}

// High degree, MG, k = 8, R_H <= 32, integer sketch values: lane-parallel
// merge in two launches.
//  k_mg_hi_scan: a warp per vertex (lane g = chunk g, register sketch) stores
//    its 32 part sketches (keys then values, physical slots) to scratch
//    indexed by worklist position, plus (cur, f0, lower_changed);
//  k_mg_hi_merge: LANE j = worklist entry j replays parts[1..] into parts[0]
//    in order through a register sketch (lpa.py:179-186, sketch.py:76-91) --
//    32 merges for the instructions of one warp-wide merge -- then the warp
//    finishes its 32 vertices (label word, dependant marks) cooperatively.
constexpr int kLpmWords = 32 * 16;  // 32 parts x (8 keys + 8 values)

template <class W, bool DET, class V>
__global__ void __launch_bounds__(SLPA_HI_THREADS, SLPA_HI_MINB) k_mg_hi_scan(SweepArgs a, const int32_t *__restrict__ list,
                                                         int64_t count, int round0) {
    static_assert(sizeof(V) == 4, "scratch holds 32-bit values");
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= count) return;  // warp-uniform
    const int32_t v = __ldg(&list[wid]);
    const uint8_t f0 = a.flag_cur[v];
    const bool act = DET ? !(round0 && !f0) : f0 != 0;
    if (!act) {
        if (lane == 0) a.hmeta[wid] = make_uint2(0u, 0u);
        return;
    }
    if (!DET) {
        __syncwarp();
        if (lane == 0) a.flag_cur[v] = 0;
    }
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
    MgSketchOff8 part;
    part.reset(8, a.zkey);
    int64_t cs = 0, ce = 0;
    if (lane < a.parts) chunk_bounds(hi - lo, a.parts, lane, cs, ce);
    bool lc = false;
    lane_stream_p<W, DET>(a, lo + cs, ce - cs, v, lc, [&](int64_t, bool valid, int32_t c, W w) {
        if (valid) part.acc(c, (V)w, 8);
    });
    const bool lca = __any_sync(0xffffffffu, lc);
    uint32_t *dst = a.hparts + (size_t)wid * kLpmWords;
    uint4 *kd = reinterpret_cast<uint4 *>(dst + lane * 8);
    uint4 *vd = reinterpret_cast<uint4 *>(dst + 256 + lane * 8);
    // streaming stores: the scratch is read once by the merge and must not
    // push the label array out of L2
    __stcs(kd, make_uint4((uint32_t)part.key[0], (uint32_t)part.key[1], (uint32_t)part.key[2], (uint32_t)part.key[3]));
    __stcs(kd + 1, make_uint4((uint32_t)part.key[4], (uint32_t)part.key[5], (uint32_t)part.key[6], (uint32_t)part.key[7]));
    __stcs(vd, make_uint4((uint32_t)part.value(0), (uint32_t)part.value(1), (uint32_t)part.value(2), (uint32_t)part.value(3)));
    __stcs(vd + 1, make_uint4((uint32_t)part.value(4), (uint32_t)part.value(5), (uint32_t)part.value(6), (uint32_t)part.value(7)));
    if (lane == 0) a.hmeta[wid] = make_uint2((uint32_t)cur, 1u | (f0 ? 2u : 0u) | (lca ? 4u : 0u));
}

template <class W, bool DET, class V>
__global__ void __launch_bounds__(kThreads, SLPA_MERGE_MINB) k_mg_hi_merge(SweepArgs a, const int32_t *__restrict__ list,
                                                          int64_t count, int) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= count) return;
    const uint2 meta = __ldcg(&a.hmeta[idx]);
    if (!(meta.y & 1u)) return;
    const uint32_t *src = a.hparts + (size_t)idx * kLpmWords;
    MgSketchOff8 S;
    S.reset(8, a.zkey);
    uint32_t kk[8], vv[8], kn[8], vn[8];
    ld8(src, kk);
    ld8(src + 256, vv);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        S.load_slot(i, (int32_t)kk[i], (V)vv[i]);
    }
    ld8(src + 8, kk);
    ld8(src + 256 + 8, vv);
    for (int q = 1; q < a.parts; ++q) {
        if (q + 1 < a.parts) {  // next part requested before this one is replayed
            ld8(src + (q + 1) * 8, kn);
            ld8(src + 256 + (q + 1) * 8, vn);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (vv[i] != 0u) S.acc((int32_t)kk[i], (V)vv[i], 8);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            kk[i] = kn[i];
            vv[i] = vn[i];
        }
    }
    int32_t best;
    const int32_t cand = S.max_key(8, best) ? best : (int32_t)meta.x;
    a.hparts[(size_t)idx * kLpmWords] = (uint32_t)cand;  // part 0's first key is no longer needed
}

// Finish of the merged vertices: a warp per entry, as k_mg_hi_direct.
template <bool DET>
__global__ void __launch_bounds__(kThreads) k_mg_hi_finish(SweepArgs a, const int32_t *__restrict__ list,
                                                           int64_t count, int) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= count) return;
    const uint2 meta = __ldcg(&a.hmeta[wid]);
    if (!(meta.y & 1u)) return;
    const int32_t v = __ldg(&list[wid]);
    const int32_t cand = (int32_t)__ldcg(&a.hparts[(size_t)wid * kLpmWords]);
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    warp_hi_finish<DET>(a, v, (int32_t)meta.x, cand, (meta.y & 2u) ? 1 : 0, (meta.y & 4u) != 0, lo, hi, lane);
}

// Group-wise chunk scan straight from the CSR: the 8 lanes of a group hold
// the 8 slots of one part sketch; lane sl loads arc x + sl of each batch
// (32-byte coalesced per group) and gathers its label, DEPTH batches ahead,
// then every arc is broadcast to the group and accumulated slot-parallel
// (first matching lane, else first empty lane, else every lane decrements).
// The per-arc chain is a few instructions and one vote -- ~5x shorter than a
// lane's register-sketch update -- which is what long chunks need.
template <class W, bool DET, class V>
__device__ __forceinline__ void group_chunk_scan(const SweepArgs &a, int64_t start, int64_t len, int64_t maxlen,
                                                 int32_t v, int sl, int gb, int32_t &key, V &val, bool &lc) {
    constexpr int D = SLPA_GCS_DEPTH;  // batches in flight (each a target load -> label gather chain)
    const W *__restrict__ wts = reinterpret_cast<const W *>(a.w);
    uint32_t Lr[D];
    W wr[D];
    auto fetch = [&](int64_t x, uint32_t &L, W &w) {
        L = 0;
        w = (W)0;
        if (x + sl < len) {
            const int32_t t = __ldg(&a.tgt[start + x + sl]);
            if (t != v) {
                w = __ldg(&wts[start + x + sl]);
                L = DET ? __ldcg(&a.lab_new[t]) : (uint32_t)__ldcg(&a.lab_old[t]);
                if (DET && t > v && (L >> 31)) L = (uint32_t)__ldg(&a.lab_old[t]);
            }
        }
    };
#pragma unroll
    for (int d = 0; d < D; ++d) fetch((int64_t)d * 8, Lr[d], wr[d]);
    for (int64_t x0 = 0; x0 < maxlen; x0 += 8 * D) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const int64_t x = x0 + d * 8;
            if (x < maxlen) {  // warp-uniform
                const uint32_t Lx = Lr[d];
                const W wx = wr[d];
                fetch(x + 8 * D, Lr[d], wr[d]);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t Lj = __shfl_sync(0xffffffffu, Lx, gb + j);
                    const W wj = __shfl_sync(0xffffffffu, wx, gb + j);
                    const bool live = x + j < len && wj != (W)0;  // group-uniform
                    lc |= live && (Lj >> 31) != 0;
                    const int32_t c = (int32_t)(Lj & SLPA_LMASK);
                    const V w = (V)wj;
                    const unsigned mm = (__ballot_sync(0xffffffffu, key_matches(key, c, a.zkey)) >> gb) & 0xffu;
                    const unsigned fm = (__ballot_sync(0xffffffffu, val == (V)0) >> gb) & 0xffu;
                    const unsigned sel = mm ? (mm & (0u - mm)) : (fm & (0u - fm));
                    const V d0 = (mm | fm) ? (V)0 : w;
                    if (live) {
                        const bool mine = (sel >> sl) & 1u;
                        if (mine) key = c;
                        val = mine ? val + w : val - (val < d0 ? val : d0);
                    }
                }
            }
        }
    }
}

// High degree, small rounds, fully fused: a block per vertex scans its 32
// chunks slot-parallel straight from the CSR (group_chunk_scan), stages the
// part sketches in shared memory, and warp 0 replays them in order on the
// slot-parallel warp sketch and finishes the vertex -- one launch and short
// chains, for rounds whose cost is latency rather than volume.
template <class W, bool DET, class V>
__global__ void __launch_bounds__(kGiantWarps * 32) k_mg_hi_block(SweepArgs a, const int32_t *__restrict__ list,
                                                                 int64_t count, int round0) {
    __shared__ int32_t s_key[32][8];
    __shared__ V s_val[32][8];
    const int64_t idx = blockIdx.x;
    if (idx >= count) return;
    const int32_t v = __ldg(&list[idx]);
    const uint8_t f0 = a.flag_cur[v];
    if (DET ? (round0 && !f0) : !f0) return;  // block-uniform
    if (!DET) {
        __syncthreads();
        if (threadIdx.x == 0) a.flag_cur[v] = 0;
    }
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int grp = lane >> 3, sl = lane & 7, gb = grp * 8;
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int64_t deg = hi - lo;
    const int P = a.parts;
    const int p = wib * 4 + grp;
    int64_t cs = 0, ce = 0;
    if (p < P) chunk_bounds(deg, P, p, cs, ce);
    int64_t maxlen = ce - cs;
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
        const int64_t x = __shfl_xor_sync(0xffffffffu, maxlen, o);
        maxlen = x > maxlen ? x : maxlen;
    }
    int32_t key = kNoKey;
    V val = (V)0;
    bool lc = false;
    group_chunk_scan<W, DET, V>(a, lo + cs, ce - cs, maxlen, v, sl, gb, key, val, lc);
    if (p < P) {
        s_key[p][sl] = key;
        s_val[p][sl] = val;
    }
    const int lc_any = __syncthreads_or(lc ? 1 : 0);
    if (wib != 0) return;
    const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
    WarpSketch<V> S_{kNoKey, (V)0, a.zkey};
    if (lane < 8) {
        S_.key = s_key[0][lane];
        S_.val = s_val[0][lane];
    }
    for (int q = 1; q < P; ++q) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const V w = s_val[q][i];
            if (w > (V)0) S_.acc(lane, 8, s_key[q][i], w);
        }
    }
    int32_t best;
    const bool found = S_.max_key(lane, 8, best);
    warp_hi_finish<DET>(a, v, cur, found ? best : cur, f0, lc_any != 0, lo, hi, lane);
}

// Low degree, small rounds: a warp per vertex.  The row's targets, weights
// and labels are loaded by all lanes at once (one round trip instead of a
// lane's chain of batches); then the arcs are replayed in adjacency order on
// the slot-parallel warp sketch (MG, physical slot rules) or on a vote every
// lane keeps redundantly (BM).  Same results as k_lane_direct; chosen when a
// round has few light vertices and its cost is latency.
template <class W, bool DET, class V, bool BM>
__global__ void __launch_bounds__(kThreads) k_lo_warp(SweepArgs a, const int32_t *__restrict__ list, int64_t count,
                                                      int round0) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= count) return;  // warp-uniform
    const int32_t v = __ldg(&list[wid]);
    const uint8_t f0 = a.flag_cur[v];
    if (DET ? (round0 && !f0) : !f0) return;
    if (!DET) {
        __syncwarp();
        if (lane == 0) a.flag_cur[v] = 0;
    }
    const W *__restrict__ wts = reinterpret_cast<const W *>(a.w);
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
    const int k = a.k;
    WarpSketch<V> S_{kNoKey, (V)0, a.zkey};
    BmVote<V> st{cur, (V)0};
    bool lc = false;
    for (int pass = 0; pass < (!BM && a.scan_double ? 2 : 1); ++pass) {
        if (pass == 1) S_.val = (V)0;  // double scan: exact re-count over the physical keys
        for (int64_t base = lo; base < hi; base += 128) {
            uint32_t L[4];
            W w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t e = base + j * 32 + lane;
                L[j] = 0;
                w[j] = (W)0;
                if (e < hi) {
                    const int32_t t = __ldg(&a.tgt[e]);
                    if (t != v) {
                        w[j] = __ldg(&wts[e]);
                        L[j] = DET ? __ldcg(&a.lab_new[t]) : (uint32_t)__ldcg(&a.lab_old[t]);
                        if (DET && t > v && (L[j] >> 31)) L[j] = (uint32_t)__ldg(&a.lab_old[t]);
                        if (DET) lc |= (L[j] >> 31) != 0;
                    }
                }
            }
            const int64_t rem = hi - base;
            const int nj = rem >= 128 ? 4 : (int)((rem + 31) / 32);
            for (int j = 0; j < nj; ++j) {
                const int ns = (int)min((int64_t)32, rem - j * 32);
                for (int src = 0; src < ns; ++src) {
                    const W wj = __shfl_sync(0xffffffffu, w[j], src);
                    const int32_t c = (int32_t)(__shfl_sync(0xffffffffu, L[j], src) & SLPA_LMASK);
                    if (wj == (W)0) continue;  // self arc (weights are > 0); warp-uniform
                    if (BM) st.acc(c, (V)wj);
                    else if (pass == 0) S_.acc(lane, k, c, (V)wj);
                    else S_.rescan_add(lane, k, c, (V)wj);
                }
            }
        }
    }
    int32_t cand = cur;
    if (BM) {
        if (hi > lo) cand = st.cand;
    } else {
        int32_t best;
        if (S_.max_key(lane, k, best)) cand = best;
    }
    warp_hi_finish<DET>(a, v, cur, cand, f0, __any_sync(0xffffffffu, lc), lo, hi, lane);
}

// High degree, BM, direct streaming.
template <class W, bool DET, class V>
__global__ void __launch_bounds__(kThreads) k_bm_hi_direct(SweepArgs a, const int32_t *__restrict__ list,
                                                           int64_t count, int round0) {
    const int lane = threadIdx.x & 31;
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
    bool lower_changed = false, have = false;
    int32_t bc = 0;
    V bw = (V)0;
    for (int p = lane; p < P; p += 32) {
        int64_t cs, ce;
        chunk_bounds(deg, P, p, cs, ce);
        BmVote<V> st{cur, (V)0};
        lane_stream_u<W, DET>(a, lo + cs, ce - cs, v, lower_changed, [&](int64_t, bool valid, int32_t c, W w) {
            if (valid) st.acc(c, (V)w);
        });
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

// ================================================================== giant vertices
// deg >= giant threshold: a single warp per vertex would walk deg/32 arcs per
// lane with dependent staging latencies on every window -- the tail of every
// heavy phase (8 ms for the 406k-degree hub at RMAT s24).  Two kernels:
//  (A) gather: a block per giant materialises its arcs' (label word, weight)
//      stream -- lower neighbours' L1|changed, higher neighbours' L0, self
//      arcs weight 0 -- coalesced and fully parallel;
//  (B) scan: a warp per giant, lane g replays chunk g from that contiguous
//      buffer with register double-buffered prefetch, so the per-lane chain
//      runs at ALU speed; then the ordered merge as in k_mg_hi_direct.
constexpr int kGatherThreads = 256;

// grid (segments, giants): block x of giant y gathers arcs
// [x * kGatherArcs, (x + 1) * kGatherArcs) of its row, 8 per thread with one
// 256-bit target load and 8 independent label gathers in flight.
constexpr int kGatherArcs = kGatherThreads * kBatch;

template <class W, bool DET>
__global__ void __launch_bounds__(kGatherThreads) k_giant_gather(SweepArgs a, const int32_t *__restrict__ slots,
                                                                 int64_t count, int round0) {
    const int64_t gi = blockIdx.y;
    if (gi >= count) return;
    const int32_t slot = __ldg(&slots[gi]);
    const int32_t v = __ldg(&a.giant_bin[slot]);
    const uint8_t f0 = a.flag_cur[v];
    if (DET ? (round0 && !f0) : !f0) return;
    const W *__restrict__ wts = reinterpret_cast<const W *>(a.w);
    W *gw = reinterpret_cast<W *>(a.gw);
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int64_t base = __ldg(&a.giant_off[slot]) - lo;
    const int64_t s0 = lo + (int64_t)blockIdx.x * kGatherArcs;
    if (s0 >= hi) return;
    const uint64_t pol = policy_evict_first();
    const int64_t e0 = s0 + (int64_t)threadIdx.x * kBatch;
    int32_t t[kBatch];
    W w[kBatch];
    uint32_t L[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
        const int64_t e = e0 + j;
        t[j] = e < hi ? ld_stream(&a.tgt[e], pol) : v;
        w[j] = e < hi ? ld_stream(&wts[e], pol) : (W)0;
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
        L[j] = 0;
        if (t[j] != v) L[j] = DET ? __ldcg(&a.lab_new[t[j]]) : (uint32_t)__ldcg(&a.lab_old[t[j]]);
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
        if (DET && t[j] > v && (L[j] >> 31)) L[j] = (uint32_t)__ldg(&a.lab_old[t[j]]);
        const int64_t e = e0 + j;
        if (e < hi) {
            __stcs(&a.glab[base + e], L[j]);  // read once by the replay: keep L2 for the labels
            __stcs(&gw[base + e], t[j] == v ? (W)0 : w[j]);
        }
    }
}

// Per-lane replay of [x, end) of a giant's gathered stream: 32-byte aligned
// 8-element batches (256-bit loads), a ring of D batches in flight so the
// per-lane sketch chain never waits on memory.  Giants are a handful of
// warps, so the ring's registers cost no occupancy that matters.
template <class W, class F>
__device__ __forceinline__ void giant_stream(const SweepArgs &a, int64_t x, int64_t end, bool &lower_changed, F &&f) {
    if (x >= end) return;
    constexpr int D = 4;
    const W *gw = reinterpret_cast<const W *>(a.gw);
    uint32_t L[D][kBatch];
    W w[D][kBatch];
    const int64_t b0 = x & ~(int64_t)(kBatch - 1);
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int64_t b = b0 + d * kBatch;
        if (b < end) {
            ld8(a.glab + b, L[d]);
            ld8_cg(gw + b, w[d]);
        }
    }
    for (int64_t b = b0; b < end; b += D * kBatch) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const int64_t bb = b + d * kBatch;
            if (bb < end) {
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    const int64_t e = bb + j;
                    if (e >= x && e < end && w[d][j] != (W)0) {
                        lower_changed |= (L[d][j] >> 31) != 0;
                        f((int32_t)(L[d][j] & SLPA_LMASK), w[d][j]);
                    }
                }
                const int64_t nb = bb + D * kBatch;
                if (nb < end) {
                    ld8(a.glab + nb, L[d]);
                    ld8_cg(gw + nb, w[d]);
                }
            }
        }
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
    WarpSketch<V> S_{a.zkey, (V)0, a.zkey};
    for (int b0 = 0; b0 < P; b0 += 32) {
        const int p = b0 + lane;
        MgSketchDev<K, V> part;
        part.reset(k, a.zkey);
        int64_t cs = 0, ce = 0;
        if (p < P) chunk_bounds(deg, P, p, cs, ce);
        giant_stream<W>(a, base + cs, base + ce, lower_changed, [&](int32_t c, W w) { part.acc(c, (V)w, k); });
        warp_merge_parts<K, V>(S_, part, b0, P, k, lane);
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

// Giant MG, k = 8, R_H <= 32: one block per giant, one 8-lane group per
// chunk (lane = slot), so every arc of a chunk is a group-wise accumulate of a
// few instructions (first matching lane, else first empty lane, else every
// lane decrements) instead of a lane's full register-sketch update: the
// per-chunk sequential chain -- the critical path of a giant -- gets ~5x
// shorter.  Then warp 0 replays parts 1.. into parts[0] in order.
template <class W, bool DET, class V>
__global__ void __launch_bounds__(kGiantWarps * 32) k_mg_giant_grp(SweepArgs a, const int32_t *__restrict__ slots,
                                                                  int64_t count, int round0) {
    __shared__ int32_t s_key[32][8];
    __shared__ V s_val[32][8];
    const int64_t gi = blockIdx.x;
    if (gi >= count) return;
    const int32_t gslot = __ldg(&slots[gi]);
    const int32_t v = __ldg(&a.giant_bin[gslot]);
    const uint8_t f0 = a.flag_cur[v];
    if (DET ? (round0 && !f0) : !f0) return;  // block-uniform
    if (!DET) {
        __syncthreads();
        if (threadIdx.x == 0) a.flag_cur[v] = 0;
    }
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int grp = lane >> 3, sl = lane & 7, gb = grp * 8;
    const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
    const int64_t deg = hi - lo;
    const int64_t base = __ldg(&a.giant_off[gslot]);
    const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
    const int P = a.parts;
    const int p = wib * 4 + grp;
    int64_t cs = 0, ce = 0;
    if (p < P) chunk_bounds(deg, P, p, cs, ce);
    const W *gw = reinterpret_cast<const W *>(a.gw);
    int64_t len = ce - cs, maxlen = len;
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
        const int64_t x = __shfl_xor_sync(0xffffffffu, maxlen, o);
        maxlen = x > maxlen ? x : maxlen;
    }
    int32_t key = kNoKey;
    V val = (V)0;
    bool lc = false;
    // ring of kGiantRing batches in flight per group: the chain consumes a
    // batch (8 dependent accumulates) in far less than one memory latency
    constexpr int kGiantRing = SLPA_GIANT_RING;
    uint32_t Lr[kGiantRing];
    W wr[kGiantRing];
#pragma unroll
    for (int d = 0; d < kGiantRing; ++d) {
        const int64_t e = (int64_t)d * 8 + sl;
        Lr[d] = e < len ? __ldcg(&a.glab[base + cs + e]) : 0u;
        wr[d] = e < len ? __ldcg(&gw[base + cs + e]) : (W)0;
    }
    for (int64_t x0 = 0; x0 < maxlen; x0 += 8 * kGiantRing) {
#pragma unroll
        for (int d = 0; d < kGiantRing; ++d) {
            const int64_t x = x0 + (int64_t)d * 8;
            if (x >= maxlen) break;  // warp-uniform
            const uint32_t Lx = Lr[d];
            const W wx = wr[d];
            const int64_t e = x + 8 * kGiantRing + sl;  // refill: the batch kGiantRing ahead
            Lr[d] = e < len ? __ldcg(&a.glab[base + cs + e]) : 0u;
            wr[d] = e < len ? __ldcg(&gw[base + cs + e]) : (W)0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t Lj = __shfl_sync(0xffffffffu, Lx, gb + j);
                const W wj = __shfl_sync(0xffffffffu, wx, gb + j);
                const bool live = x + j < len && wj != (W)0;  // group-uniform
                lc |= live && (Lj >> 31) != 0;
                const int32_t c = (int32_t)(Lj & SLPA_LMASK);
                const V w = (V)wj;
                const unsigned mm = (__ballot_sync(0xffffffffu, key_matches(key, c, a.zkey)) >> gb) & 0xffu;
                const unsigned fm = (__ballot_sync(0xffffffffu, val == (V)0) >> gb) & 0xffu;
                const unsigned sel = mm ? (mm & (0u - mm)) : (fm & (0u - fm));
                const V dd = (mm | fm) ? (V)0 : w;
                if (live) {
                    const bool mine = (sel >> sl) & 1u;
                    if (mine) key = c;
                    val = mine ? val + w : val - (val < dd ? val : dd);
                }
            }
        }
    }
    if (p < P) {
        s_key[p][sl] = key;
        s_val[p][sl] = val;
    }
    const int lc_any = __syncthreads_or(lc ? 1 : 0);
    if (wib != 0) return;
    WarpSketch<V> S_{kNoKey, (V)0, a.zkey};
    if (lane < 8) {
        S_.key = s_key[0][lane];
        S_.val = s_val[0][lane];
    }
    for (int q = 1; q < P; ++q) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const V w = s_val[q][i];
            if (w > (V)0) S_.acc(lane, 8, s_key[q][i], w);
        }
    }
    int32_t best;
    const bool found = S_.max_key(lane, 8, best);
    warp_hi_finish<DET>(a, v, cur, found ? best : cur, f0, lc_any != 0, lo, hi, lane);
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
// ------------------------------------------------------------------ exact variant
// select_label_exact (lpa.py:92-107): totals = np.bincount(labels[nb],
// weights) -- every label's weights summed in ARC order in binary64 -- then
// argmax (largest total, the smallest label on ties).  A warp per vertex
// walks the row in order, 32 arcs at a time; each arc finds its label's slot
// in the warp's open-addressing table (global scratch, xcap slots, labels
// inserted with atomicCAS); the lanes holding the same slot form a group
// (match_any) and the group's lowest lane adds the members' weights one at a
// time in lane (= arc) order, so every label's total sees exactly
// bincount's sequence of additions.  O(deg) per vertex; the table is
// cleared behind the vertex.
template <class W, bool DET>
__global__ void __launch_bounds__(kThreads) k_exact_warp(SweepArgs a, const int32_t *__restrict__ list,
                                                         int64_t count, int round0) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = a.xunits;
    if (gw >= nw) return;
    int32_t *keys = reinterpret_cast<int32_t *>(a.xs) + (size_t)gw * (size_t)a.xcap;  // this warp's region
    double *tot = a.xtot + (size_t)gw * (size_t)a.xcap;
    for (int64_t idx = gw; idx < count; idx += nw) {
        const int32_t v = __ldg(&list[idx]);
        const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
        if (hi - lo <= a.xdeg_lo || hi - lo > a.xdeg_hi) continue;  // the other launch's degree tier
        const uint8_t f0 = a.flag_cur[v];
        const bool go = DET ? (!round0 || f0) : (f0 != 0);
        if (!go) continue;  // warp-uniform
        if (!DET) {
            __syncwarp();
            if (lane == 0) a.flag_cur[v] = 0;
        }
        int64_t cap = 64;  // this vertex's table: >= 2 x degree slots, so scans and clears stay O(deg)
        while (cap < 2 * (hi - lo)) cap <<= 1;
        const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
        bool lower_changed = false;
        for (int64_t e0 = lo; e0 < hi; e0 += 32) {
            const int64_t e = e0 + lane;
            int32_t t = -1, c = -1;
            double w = 0.0;
            bool ok = false;
            if (e < hi) {
                t = __ldg(&a.tgt[e]);
                ok = t != v;
                if (ok) {
                    if (DET) {
                        const uint32_t L = gather_word<true>(a, t, v);
                        lower_changed |= (L >> 31) != 0;
                        c = (int32_t)(L & SLPA_LMASK);
                    } else {
                        c = __ldcg(&a.lab_old[t]);
                    }
                    w = arc_weight<W>(a, e);
                }
            }
            int64_t slot = -1;
            if (ok) {  // labels are non-negative; -1 marks an empty slot
                int64_t h = (int64_t)(((uint32_t)c * 2654435761u) & (uint32_t)(cap - 1));
                for (;;) {
                    const int32_t old = atomicCAS(&keys[h], -1, c);
                    if (old == -1 || old == c) break;
                    h = (h + 1) & (cap - 1);
                }
                slot = h;
            }
            const unsigned grp = __match_any_sync(0xffffffffu, slot);
            const bool leader = ok && lane == __ffs(grp) - 1;
            double acc = leader ? __ldcg(&tot[slot]) : 0.0;
            for (int b = 0; b < 32; ++b) {  // members in lane (= arc) order
                const double wb = __shfl_sync(0xffffffffu, w, b);
                if (leader && ((grp >> b) & 1u)) acc += wb;
            }
            if (leader) __stcg(&tot[slot], acc);
            __syncwarp();
        }
        // argmax over the table (largest total, smallest label on ties), then clear it
        double bw = 0.0;
        int32_t bl = 0;
        bool found = false;
        for (int64_t h = lane; h < cap; h += 32) {
            const int32_t k = __ldcg(&keys[h]);
            if (k >= 0) {
                const double x = __ldcg(&tot[h]);
                if (!found || x > bw || (x == bw && k < bl)) { bw = x; bl = k; found = true; }
                keys[h] = -1;
                tot[h] = 0.0;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ow = __shfl_xor_sync(0xffffffffu, bw, o);
            const int32_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
            const int of = __shfl_xor_sync(0xffffffffu, (int)found, o);
            if (of && (!found || ow > bw || (ow == bw && ol < bl))) { bw = ow; bl = ol; found = true; }
        }
        __syncwarp();
        const int32_t cand = found ? bl : cur;  // no neighbour other than itself: the current label
        warp_hi_finish<DET>(a, v, cur, cand, f0, lower_changed, lo, hi, lane);
    }
}

// ------------------------------------------------------------------ large k
// MgSketch with any slot count (sketch.py:17-137) for configurations the
// register / slot-parallel sketches do not cover (k > 32 with chunked rows,
// k > 64): a thread per vertex, its sketch and part sketch in global scratch
// (slot i of unit u at [i * units + u], coalesced across the warp), the
// reference's exact slot rules (first match incl. stale keys, first empty,
// clamped decrement), chunks merged in order, optional double scan.  A
// correctness path: one thread walks the whole row.
template <class V>
struct MgSketchMem {
    int32_t *key;
    V *val;
    int64_t st;  // stride between slots
    int k;
    int32_t z;   // internal value of label 0
    __device__ __forceinline__ void reset() {
        for (int i = 0; i < k; ++i) { key[i * st] = kNoKey; val[i * st] = (V)0; }
    }
    __device__ __forceinline__ void acc(int32_t c, V w) {
        for (int i = 0; i < k; ++i)
            if (key_matches(key[i * st], c, z)) { key[i * st] = c; val[i * st] += w; return; }
        for (int i = 0; i < k; ++i)
            if (val[i * st] == (V)0) { key[i * st] = c; val[i * st] = w; return; }
        for (int i = 0; i < k; ++i) val[i * st] = clamp_sub(val[i * st], w);
    }
    __device__ __forceinline__ void merge_from(const MgSketchMem &o) {  // sketch.py:76-91
        for (int i = 0; i < k; ++i) {
            const V x = o.val[i * o.st];
            if (x > (V)0) acc(o.key[i * o.st], x);
        }
    }
    __device__ __forceinline__ void clear_values() {
        for (int i = 0; i < k; ++i) val[i * st] = (V)0;
    }
    __device__ __forceinline__ void rescan_add(int32_t c, V w) {
        for (int i = 0; i < k; ++i)
            if (key_matches(key[i * st], c, z)) { key[i * st] = c; val[i * st] += w; return; }
    }
    __device__ __forceinline__ bool max_key(int32_t &out) const {
        bool found = false;
        int32_t best = 0;
        V bw = (V)0;
        for (int i = 0; i < k; ++i) {
            const V x = val[i * st];
            if (x > (V)0) {
                const int32_t c = key[i * st];
                if (!found || x > bw || (x == bw && c < best)) { best = c; bw = x; found = true; }
            }
        }
        out = best;
        return found;
    }
};

template <class W, bool DET, class V>
__global__ void __launch_bounds__(kThreads) k_mg_bigk(SweepArgs a, const int32_t *__restrict__ list, int64_t count,
                                                      int round0) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nu = a.xunits;
    if (u >= nu) return;
    const int64_t U = a.xunits;
    const int k = a.k;
    int32_t *kbase = reinterpret_cast<int32_t *>(a.xs);
    V *vbase = reinterpret_cast<V *>(a.xs + (size_t)U * (size_t)k * 2 * sizeof(int32_t));
    MgSketchMem<V> S{kbase + u, vbase + u, U, k, a.zkey};
    MgSketchMem<V> part{kbase + (int64_t)k * U + u, vbase + (int64_t)k * U + u, U, k, a.zkey};
    for (int64_t idx = u; idx < count; idx += nu) {
        const int32_t v = __ldg(&list[idx]);
        const uint8_t f0 = a.flag_cur[v];
        const bool go = DET ? (!round0 || f0) : (f0 != 0);
        if (!go) continue;
        if (!DET) a.flag_cur[v] = 0;
        const int64_t lo = __ldg(&a.off[v]), hi = __ldg(&a.off[v + 1]);
        const int64_t deg = hi - lo;
        const int32_t cur = DET ? __ldg(&a.lab_old[v]) : __ldcg(&a.lab_old[v]);
        bool lower_changed = false;
        auto label_of = [&](int32_t t) -> int32_t {
            if (!DET) return __ldcg(&a.lab_old[t]);
            const uint32_t L = gather_word<true>(a, t, v);
            lower_changed |= (L >> 31) != 0;
            return (int32_t)(L & SLPA_LMASK);
        };
        S.reset();
        if (deg < a.thr || a.single) {  // lpa.py:172-176
            for (int64_t e = lo; e < hi; ++e) {
                const int32_t t = __ldg(&a.tgt[e]);
                if (t != v) S.acc(label_of(t), (V)arc_weight<W>(a, e));
            }
        } else {  // lpa.py:177-186: parts[0] then merge(parts[1..]) in order
            for (int r = 0; r < a.parts; ++r) {
                int64_t cs, ce;
                chunk_bounds(deg, a.parts, r, cs, ce);
                MgSketchMem<V> &dst = r == 0 ? S : part;
                if (r > 0) part.reset();
                for (int64_t e = lo + cs; e < lo + ce; ++e) {
                    const int32_t t = __ldg(&a.tgt[e]);
                    if (t != v) dst.acc(label_of(t), (V)arc_weight<W>(a, e));
                }
                if (r > 0) S.merge_from(part);
            }
        }
        if (a.scan_double) {  // lpa.py:187-191
            S.clear_values();
            for (int64_t e = lo; e < hi; ++e) {
                const int32_t t = __ldg(&a.tgt[e]);
                if (t != v) S.rescan_add(label_of(t), (V)arc_weight<W>(a, e));
            }
        }
        int32_t best;
        const int32_t cand = (deg > 0 && S.max_key(best)) ? best : cur;
        unsigned long long n_delta = 0;
        if (DET) {
            const bool T = f0 || (a.symmetric ? lower_changed : lower_in_changed(a, v));
            det_commit_output(a, v, cur, cand, T, lo, hi);
        } else {
            async_commit_output(a, v, cur, cand, lo, hi, n_delta);
            if (n_delta) ctr_add(a.counters, CNT_DELTA, 1ull);
        }
        ctr_add(a.counters, CNT_EVALS, 1ull);
        ctr_add(a.counters, CNT_ARCS, (unsigned long long)deg);
    }
}

int hi_grp_mode() {
    static const int m = [] {
        const char *e = getenv("SLPA_HI_GRP");
        return e ? atoi(e) : 2;
    }();
    return m;
}

int async_split_mode() {
    static const int m = [] {
        const char *e = getenv("SLPA_ASYNC_SPLIT");
        return e ? atoi(e) : 1;
    }();
    return m;
}

int giant_grp_mode() {
    static const int m = [] {
        const char *e = getenv("SLPA_GIANT_GRP");
        return e ? atoi(e) : 1;
    }();
    return m;
}

// Kernel choice per configuration.  k = 8 with R_H <= 32 and single scan:
// scan / lane-parallel merge / finish for the deterministic high-degree
// rounds and the grouped giant kernel.  SLPA_HI_GRP=0 / SLPA_GIANT_GRP=0
// select the warp-merge kernels the other configurations use, so every
// execution path stays covered by the parity matrix (tests/test_gpu_paths.py).
template <class W, bool DET, class V>
KernelSet pick_kernels(const slpa_config *cfg) {
    if (cfg->variant == SLPA_VARIANT_EXACT) {
        KernelSet ks{k_exact_warp<W, DET>, k_exact_warp<W, DET>, k_exact_warp<W, DET>, nullptr, nullptr, kThreads,
                     kThreads, 0, 0, nullptr, nullptr, nullptr};
        ks.xmode = 1;
        return ks;
    }
    if (slpa_large_k(cfg)) {
        KernelSet ks{k_mg_bigk<W, DET, V>, k_mg_bigk<W, DET, V>, k_mg_bigk<W, DET, V>, nullptr, nullptr, kThreads,
                     kThreads, 0, 0, nullptr, nullptr, nullptr};
        ks.xmode = 2;
        return ks;
    }
    if (cfg->variant == SLPA_VARIANT_BM) {
        KernelSet ks{k_lane_direct<W, BmLane<false, V>, DET>, k_lane_direct<W, BmLane<true, V>, DET>,
                     k_bm_hi_direct<W, DET, V>, k_giant_gather<W, DET>, k_bm_giant<W, DET, V>, kThreads, kThreads, 1,
                     0, nullptr, nullptr, nullptr};
        ks.lo_small = k_lo_warp<W, DET, V, true>;
        return ks;
    }
    if (cfg->sketch_slots != 8) {
        KernelSet ks{k_lane_direct<W, MgLane<0, false, V>, DET>, k_lane_direct<W, MgLane<0, true, V>, DET>,
                     k_mg_hi_direct<W, 0, DET, V>, k_giant_gather<W, DET>, k_mg_giant<W, 0, DET, V>, kThreads,
                     kThreads, 1, 0, nullptr, nullptr, nullptr};
        if (cfg->sketch_slots <= SLPA_KHI_MAX) ks.lo_small = k_lo_warp<W, DET, V, false>;
        return ks;
    }
    const bool grouped_ok = cfg->partial_groups <= 32 && cfg->scan_mode != SLPA_SCAN_DOUBLE;
    KernelSet ks{k_lane_direct<W, MgLane<8, false, V>, DET>, k_lane_direct<W, MgLane<8, true, V>, DET>,
                 k_mg_hi_direct<W, 8, DET, V>, k_giant_gather<W, DET>, k_mg_giant<W, 8, DET, V>, kThreads, kThreads,
                 1, 0, nullptr, nullptr, nullptr};
    if constexpr (sizeof(V) == 4) {
        // async too (SLPA_ASYNC_SPLIT=0: the fused warp-merge kernel, where a
        // vertex's new label is visible to the rest of the launch at once):
        // measured 27.1 vs 29.5 ms per run at s24, communities 1.3 % vs 2.9 %
        // off the sequential count
        if (grouped_ok && hi_grp_mode() == 2 && (DET || async_split_mode())) {
            ks.hi = k_mg_hi_scan<W, DET, V>;
            ks.hi_threads = SLPA_HI_THREADS;
            ks.hi_small = k_mg_hi_block<W, DET, V>;
            ks.hi_merge = k_mg_hi_merge<W, DET, V>;
            ks.hi_finish = k_mg_hi_finish<DET>;
        }
    }
    ks.lo_small = k_lo_warp<W, DET, V, false>;
    if (grouped_ok && giant_grp_mode()) {
        ks.giant = k_mg_giant_grp<W, DET, V>;
        ks.giant_threads = kGiantWarps * 32;
    }
    return ks;
}

}  // namespace
