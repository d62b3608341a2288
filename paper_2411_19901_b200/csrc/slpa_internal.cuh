// slpa_internal.cuh -- shared declarations of the B200 label-propagation engine.
//
// Device data layout (per context, HBM):
//   CSR        off int64[n+1] | tgt int32[m] | w float32|float64[m]   (visiting order)
//   ids        int32[n]   position -> original vertex id (label value); null = identity
//   cls        uint8[n]   degree class for the current threshold (0 none, 1 low, 2 high)
//   bins       int32[n_lo] low-degree positions (ascending) | int32[n_hi] high-degree (degree desc)
//   lab_old    int32[n]   labels at the start of the sweep (L0)
//   lab_new    uint32[n]  speculative end-of-sweep labels, bit 31 = "changed" (L1 | chg<<31)
//   flag_cur   uint8[n]   unprocessed flags at the start of the sweep (F0)
//   flag_next  uint8[n]   unprocessed flags produced by this sweep (F1)
//   dirty[2]   uint32[ceil(n/32)] re-evaluation bitmaps (next round)
//   wl_lo/hi   int32[n]   round worklists
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <nvtx3/nvToolsExt.h>
#include "../../include/slpa.h"

// NVTX ranges (lpa_run / sweep / round / commit / upload) for Nsight timelines;
// header-only NVTX3, no cost without an attached tool.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

#define SLPA_CHG 0x80000000u
#define SLPA_LMASK 0x7fffffffu
#define SLPA_KDYN 64          // max sketch slots on the dynamic-k path
#define SLPA_KHI_MAX 32       // slot-parallel merge holds one slot per lane

enum { CLS_NONE = 0, CLS_LO = 1, CLS_HI = 2, CLS_MID = 3, CLS_GIANT = 4 };

struct SlpaError {
    int32_t code;
    std::string msg;
};

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            throw SlpaError{SLPA_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
    } while (0)

#define SLPA_REQUIRE(cond, code, msg) \
    do {                              \
        if (!(cond)) throw SlpaError{(code), (msg)}; \
    } while (0)

// Every device buffer carries 64 bytes of tail padding: the streaming kernels
// read arcs in 32-byte aligned batches (256-bit loads) and mask the lanes past
// the end of a row, so a batch may overhang the last arc of the array.
constexpr size_t kDevPadBytes = 64;

// Move-only owner: a throw between alloc and release (CUDA_TRY, SLPA_REQUIRE)
// frees the buffer instead of leaking it.
template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t count = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), count(o.count) { o.p = nullptr; o.count = 0; }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; count = o.count; o.p = nullptr; o.count = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t c) {
        if (c <= count && p) return;
        release();
        if (c == 0) c = 1;
        CUDA_TRY(cudaMalloc((void **)&p, c * sizeof(T) + kDevPadBytes));
        count = c;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        count = 0;
    }
    size_t bytes() const { return p ? count * sizeof(T) : 0; }
};

// Arguments shared by every sweep kernel (passed by value).
struct SweepArgs {
    const int64_t *__restrict__ off;
    const int32_t *__restrict__ tgt;
    const void *__restrict__ w;      // float or double, by template
    const int64_t *__restrict__ roff; // reverse CSR (asymmetric graphs only)
    const int32_t *__restrict__ rsrc;
    const uint8_t *__restrict__ cls;
    int32_t *lab_old;                 // det: L0 (read-only in rounds) ; async: the in-place labels
    uint32_t *lab_new;                // det only
    uint8_t *flag_cur;
    uint8_t *flag_next;
    uint32_t *dirty_next;             // det: bitmap for the next round
    unsigned long long *counters;     // [0] lo count, [1] hi count, [2] delta, [3] evals, [4] arcs
    int32_t pickless;
    int32_t k;                        // sketch slots
    int32_t parts;                    // partial_groups
    int32_t scan_double;
    int32_t symmetric;
    int32_t thr;                      // degree_threshold (chunked evaluation at deg >= thr)
    int32_t single;                   // shared_sketch: one sketch over any degree
    const int32_t *giant_bin;         // giant vertices (deg >= giant threshold), degree desc
    const int64_t *giant_off;         // exclusive prefix of their degrees
    uint32_t *glab;                   // gathered label words of their arcs
    void *gw;                         // gathered weights (W)
    uint32_t *hparts;                 // high degree, lane-parallel merge: part sketches per worklist entry
    uint2 *hmeta;                     //   (cur label, active | f0 << 1 | lower_changed << 2) per entry
    uint32_t *tbits;                  // profiling only (else null): bit v = v's last evaluation took its turn
    uint32_t *fbits;                  // det commit: next-sweep flag marks (bitmap), then written as bytes
    unsigned char *xs;                // per-unit scratch of the exact / large-k kernels (xmode != 0)
    int64_t xcap;                     //   exact: hash-table slots per warp; large k: unused
    int64_t xunits;                   //   scratch units (threads or warps) the launch may use
    double *xtot;                     //   exact: the tables' binary64 totals (keys in xs)
    int64_t xdeg_lo, xdeg_hi;         //   exact: this launch takes the vertices with xdeg_lo < degree <= xdeg_hi
    int32_t zkey;                     // internal value of label 0 (0 unless caller labels were remapped)
    int32_t ident;                    // det round 0 of lpa_run's first sweep, no visiting order: every label
                                      // still equals its vertex id and no word has a changed bit, so the
                                      // light kernels read a neighbour's label as its id (no gather)
};

enum { CNT_LO = 0, CNT_HI = 1, CNT_DELTA = 2, CNT_EVALS = 3, CNT_ARCS = 4, CNT_EVALS_HI = 5, CNT_ARCS_HI = 6, CNT_MID = 7, CNT_GIANT = 8, CNT_GPEND = 9, CNT_N = 10 };
#define CNT_STRIPES 64
#define CNT_TOTAL (CNT_N * CNT_STRIPES)

struct Csr {
    int64_t n = 0, m = 0;
    DevBuf<int64_t> off;
    DevBuf<int32_t> tgt;
    DevBuf<float> w32;
    DevBuf<double> w64;
    void release() { off.release(); tgt.release(); w32.release(); w64.release(); n = m = 0; }
    size_t bytes() const { return off.bytes() + tgt.bytes() + w32.bytes() + w64.bytes(); }
};

struct DeviceGraph {
    int64_t n = 0, m = 0;
    int32_t w_f64 = 0;
    int32_t symmetric = 1;
    int32_t has_order = 0;
    int32_t int_weights = 0;  // exactness precondition for integer sketch values
    Csr base;              // original ids (as uploaded / generated)
    Csr perm;              // visiting-order positions (has_order only)
    DevBuf<int32_t> ids;   // position -> id (has_order)
    DevBuf<int32_t> pos;   // id -> position (has_order)
    DevBuf<int64_t> roff;  // reverse CSR of the active numbering (!symmetric)
    DevBuf<int32_t> rsrc;
    // degree bins (per threshold)
    int32_t bin_thr = -1;
    int32_t bin_single = -1;  // all non-empty vertices in the low bin (exact / shared sketch)
    int32_t bin_lo_sorted = -1;
    DevBuf<uint8_t> cls;
    DevBuf<int32_t> bin_lo, bin_mid, bin_hi, bin_giant;
    DevBuf<int64_t> giant_off;  // exclusive prefix of giant degrees (n_giant + 1)
    DevBuf<int64_t> sort_k1, sort_k2, sort_small;  // binning scratch, kept across uploads
    DevBuf<int32_t> sort_v;
    int64_t n_lo = 0, n_mid = 0, n_hi = 0, n_giant = 0, giant_arcs = 0, giant_max_deg = 0;
    int64_t lo_max_deg = 0;  // largest degree in the low bin
    int64_t max_deg = -1;    // largest degree (-1: not computed for this graph)
    const Csr &act() const { return has_order ? perm : base; }
    const int64_t *off() const { return act().off.p; }
    const int32_t *tgt() const { return act().tgt.p; }
    const void *w() const { return w_f64 ? (const void *)act().w64.p : (const void *)act().w32.p; }
    size_t bytes() const {
        return base.bytes() + perm.bytes() + ids.bytes() + pos.bytes() + roff.bytes() + rsrc.bytes() + cls.bytes() +
               bin_lo.bytes() + bin_mid.bytes() + bin_hi.bytes() + bin_giant.bytes() + giant_off.bytes();
    }
    size_t csr_bytes() const { return act().bytes(); }
};

struct WorkBuffers {
    DevBuf<int32_t> lab_old;
    DevBuf<uint32_t> lab_new;
    DevBuf<uint8_t> flag_a, flag_b;
    DevBuf<uint32_t> dirty_a, dirty_b;
    DevBuf<uint32_t> dirty_g, dirty_gp;  // asynchronous giants: their marks / marks waiting for them
    DevBuf<uint8_t> dirty_bytes;  // multi-GPU deterministic: dirty marks exchanged as bytes (dense rounds)
    DevBuf<uint32_t> lab_sent;    //   the label words last published (sparse rounds send the ones that moved)
    DevBuf<int32_t> xlist;        //   this rank's sparse round list: (id, word) pairs, then remote mark ids
    DevBuf<uint32_t> tbits;       // profiling: turn bitmap (the sequential sweep's processed set)
    DevBuf<uint32_t> fbits;       // det commit: next-sweep flag bitmap
    DevBuf<unsigned long long> dcount;
    DevBuf<int32_t> wl_lo, wl_mid, wl_hi, wl_giant;
    DevBuf<uint32_t> hparts;      // lane-parallel merge scratch (high degree)
    DevBuf<uint2> hmeta;
    DevBuf<uint32_t> glab;        // giant gather buffers
    DevBuf<unsigned char> gw;
    DevBuf<int32_t> io_labels;  // staging for host <-> device label exchange
    DevBuf<uint8_t> io_flags;
    DevBuf<unsigned long long> counters;
    DevBuf<double> metric_d;    // tallies for modularity
    DevBuf<unsigned long long> metric_u;
    DevBuf<unsigned char> scratch;  // cub temp storage
    DevBuf<unsigned char> xscratch; // exact / large-k kernels: per-warp hash-table keys or per-thread sketches
    DevBuf<double> xtotals;         // exact: per-warp hash-table totals
    size_t bytes() const {
        return lab_old.bytes() + lab_new.bytes() + flag_a.bytes() + flag_b.bytes() + dirty_a.bytes() + dirty_bytes.bytes() + lab_sent.bytes() + xlist.bytes() + dirty_g.bytes() + dirty_gp.bytes() +
               dirty_b.bytes() + tbits.bytes() + fbits.bytes() + hparts.bytes() + hmeta.bytes() + wl_lo.bytes() + wl_mid.bytes() + wl_hi.bytes() + wl_giant.bytes() + glab.bytes() + gw.bytes() + io_labels.bytes() + io_flags.bytes() +
               counters.bytes() + metric_d.bytes() + metric_u.bytes() + scratch.bytes() + xscratch.bytes() + xtotals.bytes();
    }
};

struct slpa_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    DeviceGraph g;
    WorkBuffers wb;
    unsigned long long *h_counters = nullptr;  // pinned mirror of wb.counters (striped)
    int32_t *h_stage = nullptr;                // pinned staging for label downloads
    int64_t h_stage_n = 0;
    unsigned long long h_sum[CNT_N] = {};      // per-counter sums of the stripes
    std::string err;
    slpa_run_stats stats{};
    int32_t prof_on = 0;
    slpa_profile prof{};
    cudaEvent_t pev0 = nullptr, pev1 = nullptr;
    cudaStream_t stream2 = nullptr;          // giant-vertex work overlapping the main stream
    cudaEvent_t gev0 = nullptr, gev1 = nullptr;
    int32_t giant_pending = 0;
    int32_t have_labels = 0;   // lab_old holds labels of a finished run
    const slpa_config *cur_cfg = nullptr;  // configuration of the sweep being run
    // caller label values -> internal (slpa_labels_from_host): 0 identity, 1 shift, 2 rank table
    int32_t lmap_mode = 0;
    int64_t lmap_shift = 0, lmap_n = 0;
    DevBuf<int32_t> lmap_table;
    int32_t zkey = 0;  // internal value of label 0
    int32_t labels_initial = 0;  // labels are the ids lpa_run starts from (no sweep since slpa_init_labels)
    int64_t xs_key = 0, xs_units = 0;      // layout of wb.xscratch (exact table size or -k; units)
    cudaStream_t cstream = nullptr;        // host->device copies of a pipelined upload
    cudaEvent_t cev = nullptr;             //   (chunk copied)
    unsigned long long pre_checks[8] = {}; // arc checks computed during the upload (see slpa_graph_finalize)
    int32_t pre_checks_valid = 0;
    int32_t l2_saved = 0;      // set_label_l2_window changed the process's persisting set-aside
    size_t l2_prev_limit = 0;  //   ... which was this before
    // multi-GPU partition
    int32_t part = 0;
    int32_t part_sym_known = 0;  // the ranks' combined arc hashes confirmed g.symmetric
    int64_t v_begin = 0, v_end = 0;
};

// ---------------------------------------------------------------- evaluation kernel sets
typedef void (*EvalKernel)(SweepArgs, const int32_t *, int64_t, int);

// lo: one lane per vertex, one sketch; mid: one lane per vertex, R_H chunks;
// hi: one warp per vertex, lane = chunk (or thread-per-vertex for `exact`);
// giant: gather + warp-per-vertex replay.
struct KernelSet {
    EvalKernel lo, mid, hi, gather, giant;
    int lo_threads, hi_threads;
    int hi_vpw;         // hi kernel: vertices per warp (0 = one thread per vertex)
    int giant_threads;  // giant kernel: block per giant of this size (0 = warp per giant)
    EvalKernel hi_merge;   // non-null: `hi` is a scan writing part sketches, this kernel merges them
    EvalKernel hi_finish;  //   and this one (a warp per vertex) commits the merged candidates
    EvalKernel hi_small;   // small high-degree rounds: fused block-per-vertex kernel
    EvalKernel lo_small;   // small low-degree rounds: warp per vertex
    int xmode;             // 0; 1: `lo` is the exact warp-per-vertex kernel (hash table per warp);
                           // 2: `lo` is the large-k thread-per-vertex kernel (two sketches per thread)
};

// slpa_eval_<weights>_<sketch values>_<mode>.cu
KernelSet slpa_pick_f32_u32_det(const slpa_config *cfg);
KernelSet slpa_pick_f32_u32_async(const slpa_config *cfg);
KernelSet slpa_pick_f32_f64_det(const slpa_config *cfg);
KernelSet slpa_pick_f32_f64_async(const slpa_config *cfg);
KernelSet slpa_pick_f64_u32_det(const slpa_config *cfg);
KernelSet slpa_pick_f64_u32_async(const slpa_config *cfg);
KernelSet slpa_pick_f64_f64_det(const slpa_config *cfg);
KernelSet slpa_pick_f64_f64_async(const slpa_config *cfg);

// MG configurations beyond the register / warp sketches (k > 32 with chunked
// rows, or k > 64): every vertex runs the large-k kernel from the single bin.
static inline bool slpa_large_k(const slpa_config *cfg) {
    return cfg->variant == SLPA_VARIANT_MG && (cfg->shared_sketch ? cfg->sketch_slots > SLPA_KDYN
                                                                  : cfg->sketch_slots > SLPA_KHI_MAX);
}

// ---------------------------------------------------------------- host-side helpers
void slpa_validate_config(const slpa_config *cfg);
void slpa_ensure_bins(slpa_ctx *ctx, const slpa_config *cfg);
void slpa_graph_finalize(slpa_ctx *ctx);  // symmetry check, reverse CSR, reset bins
void slpa_arc_checks_range(slpa_ctx *ctx, const Csr &c, int w_f64, int64_t e0, int64_t e1, unsigned long long *acc);
void slpa_validate_arcs_range(slpa_ctx *ctx, const Csr &c, int w_f64, int64_t e0, int64_t e1, unsigned *err);
void slpa_validate_offsets_async(slpa_ctx *ctx, const Csr &c, unsigned *err);
void slpa_throw_validation(unsigned e);
void slpa_graph_apply_order(slpa_ctx *ctx, const int64_t *order_host_or_dev, bool on_device);
void slpa_alloc_work(slpa_ctx *ctx);
void slpa_assemble_unit_edges(slpa_ctx *ctx, int64_t n, int64_t num_edges, uint32_t *d_src, uint32_t *d_dst);

// sweep drivers (slpa_sweep.cu)
int64_t slpa_sweep_det(slpa_ctx *ctx, const slpa_config *cfg, int pickless);
int64_t slpa_sweep_async(slpa_ctx *ctx, const slpa_config *cfg, int pickless);
void slpa_part_det_round_impl(slpa_ctx *ctx, const slpa_config *cfg, int pickless, int round);
int64_t slpa_part_det_import_impl(slpa_ctx *ctx);
void slpa_part_det_collect_impl(slpa_ctx *ctx, uint64_t *list_dptr, int64_t *n_words, int64_t *n_marks);
int64_t slpa_part_det_apply_impl(slpa_ctx *ctx, const int32_t *recv, int64_t stride, const int64_t *counts_host,
                                 int32_t world, int32_t self);
void slpa_part_det_dense_impl(slpa_ctx *ctx);
int64_t slpa_part_det_commit_impl(slpa_ctx *ctx, const slpa_config *cfg);
void slpa_init_labels(slpa_ctx *ctx);  // lab = ids (or arange), flags = 1
void slpa_labels_to_host(slpa_ctx *ctx, int32_t *host);       // by original id
void slpa_labels_from_host(slpa_ctx *ctx, const int32_t *host);
void slpa_flags_to_host(slpa_ctx *ctx, uint8_t *host);
void slpa_flags_from_host(slpa_ctx *ctx, const uint8_t *host);
void slpa_permute_id_to_pos(slpa_ctx *ctx, const int32_t *d_by_id, int32_t *d_by_pos);

// metrics (slpa_metrics.cu)
void slpa_tally(slpa_ctx *ctx, const int32_t *d_labels_by_pos, double *q, int64_t *ncomm, int64_t *sizes,
                double *internal, double *incident);

static inline unsigned grid_for(int64_t count, int threads) {
    int64_t b = (count + threads - 1) / threads;
    if (b < 1) b = 1;
    return (unsigned)b;
}
