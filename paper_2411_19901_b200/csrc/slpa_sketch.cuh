// slpa_sketch.cuh -- register-resident weighted Misra-Gries sketch and weighted
// Boyer-Moore vote, with exactly the reference's slot rules and binary64
// arithmetic (sketch.py:17-181), plus the warp-cooperative slot-parallel
// merge used by the high-degree path.
#pragma once
#include "slpa_internal.cuh"

template <int K>
struct KArr {
    static constexpr int v = K > 0 ? K : SLPA_KDYN;
};

// MgSketch (sketch.py:17-137).  K > 0: compile-time slots (registers);
// K == 0: runtime k <= SLPA_KDYN (local memory).
template <int K>
struct MgSketchDev {
    int32_t key[KArr<K>::v];
    double val[KArr<K>::v];

    __device__ __forceinline__ void reset(int k) {  // MgSketch.__init__ sketch.py:34-39
        if constexpr (K > 0) {
#pragma unroll
            for (int i = 0; i < K; ++i) { key[i] = 0; val[i] = 0.0; }
        } else {
            for (int i = 0; i < k; ++i) { key[i] = 0; val[i] = 0.0; }
        }
    }

    // accumulate (sketch.py:47-74): first slot whose key equals c (stale keys
    // included) gains w; else the first slot with value 0.0 takes (c, w); else
    // every slot loses w, clamped at 0.
    __device__ __forceinline__ void acc(int32_t c, double w, int k) {
        if constexpr (K > 0) {
            int hit = -1, fr = -1;
#pragma unroll
            for (int i = K - 1; i >= 0; --i) {
                if (key[i] == c) hit = i;
                if (val[i] == 0.0) fr = i;
            }
            if (hit >= 0) {
#pragma unroll
                for (int i = 0; i < K; ++i)
                    if (i == hit) val[i] += w;
            } else if (fr >= 0) {
#pragma unroll
                for (int i = 0; i < K; ++i)
                    if (i == fr) { key[i] = c; val[i] = w; }
            } else {
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    double t = val[i] - w;
                    val[i] = t > 0.0 ? t : 0.0;
                }
            }
        } else {
            for (int i = 0; i < k; ++i)
                if (key[i] == c) { val[i] += w; return; }
            for (int i = 0; i < k; ++i)
                if (val[i] == 0.0) { key[i] = c; val[i] = w; return; }
            for (int i = 0; i < k; ++i) {
                double t = val[i] - w;
                val[i] = t > 0.0 ? t : 0.0;
            }
        }
    }

    __device__ __forceinline__ void clear_values(int k) {  // sketch.py:107-111
        if constexpr (K > 0) {
#pragma unroll
            for (int i = 0; i < K; ++i) val[i] = 0.0;
        } else {
            for (int i = 0; i < k; ++i) val[i] = 0.0;
        }
    }

    __device__ __forceinline__ void rescan_add(int32_t c, double w, int k) {  // sketch.py:113-126
        if constexpr (K > 0) {
            int hit = -1;
#pragma unroll
            for (int i = K - 1; i >= 0; --i)
                if (key[i] == c) hit = i;
#pragma unroll
            for (int i = 0; i < K; ++i)
                if (i == hit) val[i] += w;
        } else {
            for (int i = 0; i < k; ++i)
                if (key[i] == c) { val[i] += w; return; }
        }
    }

    // max_key (sketch.py:93-105): largest value, ties to the smaller key, skip v <= 0.
    __device__ __forceinline__ bool max_key(int k, int32_t &out) const {
        bool found = false;
        int32_t best = 0;
        double bw = 0.0;
        const int kk = K > 0 ? K : k;
#pragma unroll
        for (int i = 0; i < KArr<K>::v; ++i) {
            if (K == 0 && i >= kk) break;
            double v = val[i];
            if (v > 0.0) {
                int32_t c = key[i];
                if (!found || v > bw || (v == bw && c < best)) { best = c; bw = v; found = true; }
            }
        }
        out = best;
        return found;
    }
};

// BmState (sketch.py:140-162)
struct BmVote {
    int32_t cand;
    double w;
    __device__ __forceinline__ void acc(int32_t c, double x) {
        if (c == cand) w += x;
        else if (w > x) w -= x;
        else { cand = c; w = x; }
    }
};

// reduce_votes order (sketch.py:165-181): max weight, ties to smaller candidate.
__device__ __forceinline__ bool bm_better(double w1, int32_t c1, double w0, int32_t c0) {
    return w1 > w0 || (w1 == w0 && c1 < c0);
}

// _chunk_bounds (lpa.py:110-118): chunk r of `count` split into `parts`.
__device__ __forceinline__ void chunk_bounds(int64_t count, int64_t parts, int64_t r, int64_t &s, int64_t &e) {
    int64_t base = count / parts, rem = count % parts;
    s = r * base + (r < rem ? r : rem);
    e = s + base + (r < rem ? 1 : 0);
}

// ---------------------------------------------------------------- slot-parallel sketch
// The merged sketch of the high-degree path lives one slot per lane
// (lane l < k holds slot l).  `acc` replays MgSketch.accumulate with the
// physical slot rules: first matching lane (ballot + ffs), else first empty
// lane, else every lane decrements.  (c, w) must be warp-uniform.
struct WarpSketch {
    int32_t key;
    double val;
    __device__ __forceinline__ void acc(int lane, int k, int32_t c, double w) {
        const bool live = lane < k;
        unsigned mm = __ballot_sync(0xffffffffu, live && key == c);
        if (mm) {
            if (lane == __ffs(mm) - 1) val += w;
            return;
        }
        unsigned fm = __ballot_sync(0xffffffffu, live && val == 0.0);
        if (fm) {
            if (lane == __ffs(fm) - 1) { key = c; val = w; }
            return;
        }
        if (live) {
            double t = val - w;
            val = t > 0.0 ? t : 0.0;
        }
    }
    __device__ __forceinline__ void rescan_add(int lane, int k, int32_t c, double w) {
        unsigned mm = __ballot_sync(0xffffffffu, lane < k && key == c);
        if (mm && lane == __ffs(mm) - 1) val += w;
    }
    // max_key over the lanes; result valid on every lane.
    __device__ __forceinline__ bool max_key(int lane, int k, int32_t &out) const {
        double bw = (lane < k && val > 0.0) ? val : -1.0;
        int32_t bk = key;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double ow = __shfl_xor_sync(0xffffffffu, bw, o);
            int32_t ok = __shfl_xor_sync(0xffffffffu, bk, o);
            if (ow > bw || (ow == bw && ok < bk)) { bw = ow; bk = ok; }
        }
        out = bk;
        return bw > 0.0;
    }
};
