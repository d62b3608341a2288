// slpa_sketch.cuh -- register-resident weighted Misra-Gries sketch and weighted
// Boyer-Moore vote, with exactly the reference's slot rules (sketch.py:17-181),
// plus the warp-cooperative slot-parallel merge of the high-degree path.
//
// Value type V:
//   double   -- the reference's binary64 arithmetic, any positive weights;
//   uint32_t -- used only when every weight is an integer and every weighted
//               degree is < 2^31 (checked on the device at upload).  Then every
//               sketch / vote value is an integer in [0, weighted degree], so
//               binary64 add / subtract / compare are exact and the integer
//               sketch is bit-identical -- with a shorter
//               dependency chain and half the value registers.
#pragma once
#include "slpa_internal.cuh"

template <int K>
struct KArr {
    static constexpr int v = K > 0 ? K : SLPA_KDYN;
};

template <class V>
__device__ __forceinline__ V clamp_sub(V v, V w) {  // max(v - w, 0) as sketch.py:73
    if constexpr (sizeof(V) == 4) return v > w ? v - w : (V)0;
    else {
        V t = v - w;
        return t > (V)0 ? t : (V)0;
    }
}

// Key representation.  The reference initialises every key to 0
// (sketch.py:38) and matches "the first slot whose key equals c, even if
// empty" (sketch.py:59-65).  A key enters a slot only when no slot holds it,
// so every key other than the initial 0 occupies at most one slot.  Here a
// never-written slot holds kNoKey (< 0, never a label) instead of 0, which
// makes every stored key unique: an arc with label c != 0 matches at most one
// slot and needs no "first of several" resolution.  Label 0 matches the
// first slot holding 0 or kNoKey -- exactly the slots holding 0 in the
// reference -- on a (rare) slow path.  Values, stale keys, slot positions and
// therefore merge replay order, max_key and the double-scan re-count are
// identical to the reference's.
constexpr int32_t kNoKey = -1;

__device__ __forceinline__ bool key_matches(int32_t key, int32_t c) { return key == c || (c == 0 && key < 0); }

// MgSketch (sketch.py:17-137).  K > 0: compile-time slots (registers);
// K == 0: runtime k <= SLPA_KDYN (local memory).
template <int K, class V = double>
struct MgSketchDev {
    int32_t key[KArr<K>::v];
    V val[KArr<K>::v];

    __device__ __forceinline__ void reset(int k) {  // MgSketch.__init__ sketch.py:34-39
        if constexpr (K > 0) {
#pragma unroll
            for (int i = 0; i < K; ++i) { key[i] = kNoKey; val[i] = (V)0; }
        } else {
            for (int i = 0; i < k; ++i) { key[i] = kNoKey; val[i] = (V)0; }
        }
    }

    // accumulate (sketch.py:47-74): first slot whose key equals c (stale keys
    // included) gains w; else the first slot with value 0 takes (c, w); else
    // every slot loses w, clamped at 0.
    __device__ __forceinline__ void acc(int32_t c, V w, int k) {
        if constexpr (K > 0) {
            if (c != 0) {
                // fast path: the key is unique, so "first match" is "the match"
                bool any = false;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                    const bool h = key[i] == c;
                    if (h) val[i] += w;
                    any |= h;
                }
                if (any) return;
                unsigned fm = 0;
#pragma unroll
                for (int i = 0; i < K; ++i) fm |= val[i] == (V)0 ? (1u << i) : 0u;
                if (fm) {
                    const unsigned sel = fm & (0u - fm);
#pragma unroll
                    for (int i = 0; i < K; ++i)
                        if (sel & (1u << i)) { key[i] = c; val[i] = w; }
                } else {
#pragma unroll
                    for (int i = 0; i < K; ++i) val[i] = clamp_sub(val[i], w);
                }
                return;
            }
            unsigned mm = 0, fm = 0;
#pragma unroll
            for (int i = 0; i < K; ++i) {
                mm |= key_matches(key[i], c) ? (1u << i) : 0u;
                fm |= val[i] == (V)0 ? (1u << i) : 0u;
            }
            if (mm) {
                const unsigned sel = mm & (0u - mm);
#pragma unroll
                for (int i = 0; i < K; ++i)
                    if (sel & (1u << i)) { key[i] = c; val[i] += w; }
            } else if (fm) {
                const unsigned sel = fm & (0u - fm);
#pragma unroll
                for (int i = 0; i < K; ++i)
                    if (sel & (1u << i)) { key[i] = c; val[i] = w; }
            } else {
#pragma unroll
                for (int i = 0; i < K; ++i) val[i] = clamp_sub(val[i], w);
            }
        } else {
            for (int i = 0; i < k; ++i)
                if (key_matches(key[i], c)) { key[i] = c; val[i] += w; return; }
            for (int i = 0; i < k; ++i)
                if (val[i] == (V)0) { key[i] = c; val[i] = w; return; }
            for (int i = 0; i < k; ++i) val[i] = clamp_sub(val[i], w);
        }
    }

    __device__ __forceinline__ void clear_values(int k) {  // sketch.py:107-111
        if constexpr (K > 0) {
#pragma unroll
            for (int i = 0; i < K; ++i) val[i] = (V)0;
        } else {
            for (int i = 0; i < k; ++i) val[i] = (V)0;
        }
    }

    // rescan_add (sketch.py:113-126): first slot whose key equals c gains w.
    // The slot keeps kNoKey when c == 0 (values only are re-counted).
    __device__ __forceinline__ void rescan_add(int32_t c, V w, int k) {
        if constexpr (K > 0) {
            unsigned mm = 0;
#pragma unroll
            for (int i = 0; i < K; ++i) mm |= key_matches(key[i], c) ? (1u << i) : 0u;
            const unsigned sel = mm & (0u - mm);
#pragma unroll
            for (int i = 0; i < K; ++i)
                if (sel & (1u << i)) { key[i] = c; val[i] += w; }
        } else {
            for (int i = 0; i < k; ++i)
                if (key_matches(key[i], c)) { key[i] = c; val[i] += w; return; }
        }
    }

    // max_key (sketch.py:93-105): largest value, ties to the smaller key, skip v <= 0.
    __device__ __forceinline__ bool max_key(int k, int32_t &out) const {
        bool found = false;
        int32_t best = 0;
        V bw = (V)0;
        const int kk = K > 0 ? K : k;
#pragma unroll
        for (int i = 0; i < KArr<K>::v; ++i) {
            if (K == 0 && i >= kk) break;
            V v = val[i];
            if (v > (V)0) {
                int32_t c = key[i];
                if (!found || v > bw || (v == bw && c < best)) { best = c; bw = v; found = true; }
            }
        }
        out = best;
        return found;
    }
};

// BmState (sketch.py:140-162)
template <class V = double>
struct BmVote {
    int32_t cand;
    V w;
    __device__ __forceinline__ void acc(int32_t c, V x) {
        if (c == cand) w += x;
        else if (w > x) w -= x;
        else { cand = c; w = x; }
    }
};

// reduce_votes order (sketch.py:165-181): max weight, ties to smaller candidate.
template <class V>
__device__ __forceinline__ bool bm_better(V w1, int32_t c1, V w0, int32_t c0) {
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
template <class V = double>
struct WarpSketch {
    int32_t key;
    V val;
    __device__ __forceinline__ void acc(int lane, int k, int32_t c, V w) {
        const bool live = lane < k;
        const unsigned mm = __ballot_sync(0xffffffffu, live && key_matches(key, c));
        const unsigned fm = __ballot_sync(0xffffffffu, live && val == (V)0);
        if (mm) {
            if (lane == __ffs(mm) - 1) { key = c; val += w; }
        } else if (fm) {
            if (lane == __ffs(fm) - 1) { key = c; val = w; }
        } else if (live) {
            val = clamp_sub(val, w);
        }
    }
    __device__ __forceinline__ void rescan_add(int lane, int k, int32_t c, V w) {
        unsigned mm = __ballot_sync(0xffffffffu, lane < k && key_matches(key, c));
        if (mm && lane == __ffs(mm) - 1) { key = c; val += w; }
    }
    // max_key over the lanes; result valid on every lane.
    __device__ __forceinline__ bool max_key(int lane, int k, int32_t &out) const {
        const bool have = lane < k && val > (V)0;
        V bw = have ? val : (V)0;
        int32_t bk = key;
        int hv = have;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            V ow = __shfl_xor_sync(0xffffffffu, bw, o);
            int32_t ok = __shfl_xor_sync(0xffffffffu, bk, o);
            int oh = __shfl_xor_sync(0xffffffffu, hv, o);
            if (oh && (!hv || ow > bw || (ow == bw && ok < bk))) { bw = ow; bk = ok; hv = 1; }
        }
        out = bk;
        return hv != 0;
    }
};
