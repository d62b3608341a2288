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

// z: the internal value of label 0 -- 0, unless caller labels were remapped
// (negative labels, slpa_labels_from_host), when it is the image of 0.
__device__ __forceinline__ bool key_matches(int32_t key, int32_t c, int32_t z) { return key == c || (c == z && key < 0); }

// MgSketch (sketch.py:17-137).  K > 0: compile-time slots (registers);
// K == 0: runtime k <= SLPA_KDYN (local memory).
template <int K, class V = double>
struct MgSketchDev {
    int32_t key[KArr<K>::v];
    V val[KArr<K>::v];
    int32_t z;  // internal value of label 0 (key_matches)

    __device__ __forceinline__ void reset(int k, int32_t z_ = 0) {  // MgSketch.__init__ sketch.py:34-39
        z = z_;
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
            if (c != z) {
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
                mm |= key_matches(key[i], c, z) ? (1u << i) : 0u;
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
                if (key_matches(key[i], c, z)) { key[i] = c; val[i] += w; return; }
            for (int i = 0; i < k; ++i)
                if (val[i] == (V)0) { key[i] = c; val[i] = w; return; }
            for (int i = 0; i < k; ++i) val[i] = clamp_sub(val[i], w);
        }
    }

    // slot i's value / load a slot (fresh sketch) / canonical form (no-op here)
    __device__ __forceinline__ V value(int i) const { return val[i]; }
    __device__ __forceinline__ void load_slot(int i, int32_t kk, V vv) { key[i] = kk; val[i] = vv; }
    __device__ __forceinline__ void normalize() {}

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
            for (int i = 0; i < K; ++i) mm |= key_matches(key[i], c, z) ? (1u << i) : 0u;
            const unsigned sel = mm & (0u - mm);
#pragma unroll
            for (int i = 0; i < K; ++i)
                if (sel & (1u << i)) { key[i] = c; val[i] += w; }
        } else {
            for (int i = 0; i < k; ++i)
                if (key_matches(key[i], c, z)) { key[i] = c; val[i] += w; return; }
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

// ---------------------------------------------------------------- integer, k = 8
// The hot sketch: 8 slots with uint32 values (exact under the integer-value
// precondition above), branch-free, in the reference's own key
// representation (every key starts at 0, sketch.py:38).
//
// Offset form.  The decrement "every slot loses w, clamped at 0"
// (sketch.py:71-74) touches all slots; here it is one add: slot i stores
// s[i] and its value is max(s[i] - D, 0), so the decrement is D += w and a
// slot is empty exactly when s[i] <= D.  A hit on slot i makes its value
// value + w, i.e. s[i] = max(s[i], D) + w = max(s[i] + w, D + w) (an empty
// slot with a stale matching key restarts at w, as values[s] += w on 0.0);
// an insert writes (c, D + w).  Every quantity stays below the vertex's
// weighted degree (< 2^31), so nothing wraps.
//
// First-match.  keys.index(c) (sketch.py:59-65) is the FIRST slot holding
// c; with keys starting at 0 label 0 may sit in several slots.  The hit
// chain carries "no earlier slot matched" in a predicate, so exactly the
// first matching slot is updated; the insert chain does the same for
// "first slot with value 0" (sketch.py:66-70).  One accumulate is ~60
// predicated instructions and no branches, so the lanes of a warp never
// diverge on hit / insert / decrement.
template <>
struct MgSketchDev<8, uint32_t> {
    int32_t key[8];
    uint32_t s[8];
    uint32_t D;

    __device__ __forceinline__ void reset(int, int32_t z = 0) {  // MgSketch.__init__ sketch.py:34-39
#pragma unroll
        for (int i = 0; i < 8; ++i) { key[i] = z; s[i] = 0u; }  // every key starts as label 0
        D = 0u;
    }
    __device__ __forceinline__ uint32_t value(int i) const { return s[i] > D ? s[i] - D : 0u; }
    __device__ __forceinline__ void load_slot(int i, int32_t kk, uint32_t vv) { key[i] = kk; s[i] = vv + D; }
    __device__ __forceinline__ void normalize() {  // D = 0 form (values stored as-is)
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = value(i);
        D = 0u;
    }

    // accumulate (sketch.py:47-74)
    __device__ __forceinline__ void acc(int32_t c, uint32_t w, int) {
        asm("{\n\t"
            ".reg .pred a, h;\n\t"
            ".reg .u32 dw, t;\n\t"
            "add.u32 dw, %16, %18;\n\t"
            "setp.ne.s32 a|h, %0, %17;\n\t"
            "@h add.u32 t, %8, %18;\n\t @h max.u32 %8, t, dw;\n\t"
            "setp.ne.and.s32 a|h, %1, %17, a;\n\t"
            "@h add.u32 t, %9, %18;\n\t @h max.u32 %9, t, dw;\n\t"
            "setp.ne.and.s32 a|h, %2, %17, a;\n\t"
            "@h add.u32 t, %10, %18;\n\t @h max.u32 %10, t, dw;\n\t"
            "setp.ne.and.s32 a|h, %3, %17, a;\n\t"
            "@h add.u32 t, %11, %18;\n\t @h max.u32 %11, t, dw;\n\t"
            "setp.ne.and.s32 a|h, %4, %17, a;\n\t"
            "@h add.u32 t, %12, %18;\n\t @h max.u32 %12, t, dw;\n\t"
            "setp.ne.and.s32 a|h, %5, %17, a;\n\t"
            "@h add.u32 t, %13, %18;\n\t @h max.u32 %13, t, dw;\n\t"
            "setp.ne.and.s32 a|h, %6, %17, a;\n\t"
            "@h add.u32 t, %14, %18;\n\t @h max.u32 %14, t, dw;\n\t"
            "setp.ne.and.s32 a|h, %7, %17, a;\n\t"
            "@h add.u32 t, %15, %18;\n\t @h max.u32 %15, t, dw;\n\t"
            // no hit (a): the first empty slot (s <= D) takes (c, D + w)
            "setp.gt.and.u32 a|h, %8, %16, a;\n\t @h mov.u32 %0, %17;\n\t @h mov.u32 %8, dw;\n\t"
            "setp.gt.and.u32 a|h, %9, %16, a;\n\t @h mov.u32 %1, %17;\n\t @h mov.u32 %9, dw;\n\t"
            "setp.gt.and.u32 a|h, %10, %16, a;\n\t @h mov.u32 %2, %17;\n\t @h mov.u32 %10, dw;\n\t"
            "setp.gt.and.u32 a|h, %11, %16, a;\n\t @h mov.u32 %3, %17;\n\t @h mov.u32 %11, dw;\n\t"
            "setp.gt.and.u32 a|h, %12, %16, a;\n\t @h mov.u32 %4, %17;\n\t @h mov.u32 %12, dw;\n\t"
            "setp.gt.and.u32 a|h, %13, %16, a;\n\t @h mov.u32 %5, %17;\n\t @h mov.u32 %13, dw;\n\t"
            "setp.gt.and.u32 a|h, %14, %16, a;\n\t @h mov.u32 %6, %17;\n\t @h mov.u32 %14, dw;\n\t"
            "setp.gt.and.u32 a|h, %15, %16, a;\n\t @h mov.u32 %7, %17;\n\t @h mov.u32 %15, dw;\n\t"
            // no hit, no empty slot: every slot loses w (the offset grows)
            "@a mov.u32 %16, dw;\n\t"
            "}"
            : "+r"(key[0]), "+r"(key[1]), "+r"(key[2]), "+r"(key[3]), "+r"(key[4]), "+r"(key[5]), "+r"(key[6]),
              "+r"(key[7]), "+r"(s[0]), "+r"(s[1]), "+r"(s[2]), "+r"(s[3]), "+r"(s[4]), "+r"(s[5]), "+r"(s[6]),
              "+r"(s[7]), "+r"(D)
            : "r"(c), "r"(w));
    }

    __device__ __forceinline__ void clear_values(int) {  // sketch.py:107-111
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = 0u;
        D = 0u;
    }

    // rescan_add (sketch.py:113-126): the first slot whose key equals c gains w
    // (after clear_values D == 0, so max(s + w, D + w) == s + w).
    __device__ __forceinline__ void rescan_add(int32_t c, uint32_t w, int) {
        asm("{\n\t"
            ".reg .pred a, h;\n\t"
            "setp.ne.s32 a|h, %8, %16;\n\t @h add.u32 %0, %0, %17;\n\t"
            "setp.ne.and.s32 a|h, %9, %16, a;\n\t @h add.u32 %1, %1, %17;\n\t"
            "setp.ne.and.s32 a|h, %10, %16, a;\n\t @h add.u32 %2, %2, %17;\n\t"
            "setp.ne.and.s32 a|h, %11, %16, a;\n\t @h add.u32 %3, %3, %17;\n\t"
            "setp.ne.and.s32 a|h, %12, %16, a;\n\t @h add.u32 %4, %4, %17;\n\t"
            "setp.ne.and.s32 a|h, %13, %16, a;\n\t @h add.u32 %5, %5, %17;\n\t"
            "setp.ne.and.s32 a|h, %14, %16, a;\n\t @h add.u32 %6, %6, %17;\n\t"
            "setp.ne.and.s32 a|h, %15, %16, a;\n\t @h add.u32 %7, %7, %17;\n\t"
            "}"
            : "+r"(s[0]), "+r"(s[1]), "+r"(s[2]), "+r"(s[3]), "+r"(s[4]), "+r"(s[5]), "+r"(s[6]), "+r"(s[7])
            : "r"(key[0]), "r"(key[1]), "r"(key[2]), "r"(key[3]), "r"(key[4]), "r"(key[5]), "r"(key[6]),
              "r"(key[7]), "r"(c), "r"(w));
    }

    // max_key (sketch.py:93-105): largest value, ties to the smaller key, skip v <= 0.
    __device__ __forceinline__ bool max_key(int, int32_t &out) const {
        bool found = false;
        int32_t best = 0;
        uint32_t bw = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t v = value(i);
            if (v > 0u) {
                const int32_t c = key[i];
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
    int32_t z;  // internal value of label 0
    __device__ __forceinline__ void acc(int lane, int k, int32_t c, V w) {
        const bool live = lane < k;
        const unsigned mm = __ballot_sync(0xffffffffu, live && key_matches(key, c, z));
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
        unsigned mm = __ballot_sync(0xffffffffu, lane < k && key_matches(key, c, z));
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
