// slpa_part.cu -- multi-GPU: one context per rank holds the rows of a
// contiguous vertex range [v_begin, v_end).
//
// The rank's CSR keeps the global numbering: offsets has n+1 entries with
// empty rows outside the range, targets are global ids.  Every sweep kernel
// therefore runs unchanged on the owned rows.  labels (lab_old) is a full
// replica; flags is global-sized too: owned entries are this rank's
// unprocessed flags, remote entries collect the marks this rank's changed
// vertices send to their neighbours (lpa.py:223).  Between sweeps the host
// all-gathers the owned label ranges and max-reduces the flag arrays over
// NCCL (paper_2411_19901_b200/distributed.py); slpa_part_end_exchange then
// clears the remote entries again.  Execution is the asynchronous sweep
// (remote labels are one exchange old), as in the paper's multi-GPU model.
#include <algorithm>
#include "slpa_internal.cuh"

void slpa_graph_validate(slpa_ctx *ctx, const Csr &c, int w_f64);
void slpa_check_int_weights(slpa_ctx *ctx);
void slpa_part_gen_rmat_impl(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB,
                             uint32_t tABC, uint64_t seed, int32_t permute, uint64_t perm_key, int64_t r0,
                             int64_t r1);
void slpa_part_tally_impl(slpa_ctx *ctx, double *internal_local, uint64_t *incident_dptr, uint64_t *sizes_dptr);
void slpa_arc_hash_impl(slpa_ctx *ctx, uint64_t out[4]);
void slpa_rmat_cuts_impl(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB, uint32_t tABC,
                         uint64_t seed, int32_t permute, uint64_t perm_key, int32_t world, int64_t *cuts_out);
void slpa_part_modularity_impl(slpa_ctx *ctx, double internal_total, double *q);

namespace {
__global__ void k_part_offsets(const int64_t *loc, int64_t n, int64_t vb, int64_t ve, int64_t mloc, int64_t *off) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v > n) return;
    off[v] = v <= vb ? 0 : (v >= ve ? mloc : loc[v - vb]);
}

template <class F>
int32_t guard(slpa_ctx *ctx, F &&f) {
    try {
        ctx->err.clear();
        cudaError_t e = cudaSetDevice(ctx->device);
        if (e != cudaSuccess) throw SlpaError{SLPA_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)};
        f();
        return SLPA_OK;
    } catch (const SlpaError &e) {
        ctx->err = e.msg;
        return e.code;
    } catch (const std::exception &e) {
        ctx->err = e.what();
        return SLPA_ECUDA;
    }
}

void mark_partitioned(slpa_ctx *ctx, int64_t vb, int64_t ve) {
    DeviceGraph &g = ctx->g;
    ctx->part = 1;
    ctx->v_begin = vb;
    ctx->v_end = ve;
    g.perm.release();
    g.ids.release();
    g.pos.release();
    g.has_order = 0;
    g.roff.release();
    g.rsrc.release();
    // Symmetry is a property of the whole graph: unknown until the ranks
    // combine their arc hashes (slpa_part_arc_hash -> slpa_part_set_symmetric).
    // The asynchronous sweep does not depend on it; the deterministic rounds
    // require it (their dependant marks follow out-arcs).
    g.symmetric = 0;
    ctx->part_sym_known = 0;
    slpa_check_int_weights(ctx);
    g.max_deg = -1;
    g.bin_thr = -1;
    g.bin_single = -1;
    g.bin_lo_sorted = -1;
    ctx->have_labels = 0;
}

void require_part(slpa_ctx *ctx) {
    SLPA_REQUIRE(ctx->part && ctx->g.base.off.p, SLPA_ENOGRAPH, "no partition resident");
}
}  // namespace

extern "C" {

int32_t slpa_part_upload(slpa_ctx *ctx, int64_t n, int64_t v_begin, int64_t v_end, const int64_t *row_offsets,
                         const int32_t *targets, const void *weights, int32_t weights_f64) {
    return guard(ctx, [&] {
        SLPA_REQUIRE(n >= 0 && n < (1LL << 31) - 1, SLPA_EINVAL, "bad vertex count");
        SLPA_REQUIRE(v_begin >= 0 && v_begin <= v_end && v_end <= n, SLPA_EINVAL, "bad vertex range");
        DeviceGraph &g = ctx->g;
        cudaStream_t s = ctx->stream;
        const int64_t nloc = v_end - v_begin;
        const int64_t mloc = row_offsets[nloc];
        SLPA_REQUIRE(row_offsets[0] == 0 && mloc >= 0, SLPA_EINVAL, "row offsets must start at 0");
        g.base.release();
        g.base.n = n;
        g.base.m = mloc;
        g.base.off.alloc(n + 1);
        g.base.tgt.alloc(mloc);
        DevBuf<int64_t> loc;
        loc.alloc(nloc + 1);
        CUDA_TRY(cudaMemcpyAsync(loc.p, row_offsets, (nloc + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        k_part_offsets<<<grid_for(n + 1, 256), 256, 0, s>>>(loc.p, n, v_begin, v_end, mloc, g.base.off.p);
        CUDA_TRY(cudaGetLastError());
        if (mloc) CUDA_TRY(cudaMemcpyAsync(g.base.tgt.p, targets, mloc * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        if (weights_f64) {
            g.base.w64.alloc(mloc);
            if (mloc) CUDA_TRY(cudaMemcpyAsync(g.base.w64.p, weights, mloc * sizeof(double), cudaMemcpyHostToDevice, s));
        } else {
            g.base.w32.alloc(mloc);
            if (mloc) CUDA_TRY(cudaMemcpyAsync(g.base.w32.p, weights, mloc * sizeof(float), cudaMemcpyHostToDevice, s));
        }
        CUDA_TRY(cudaStreamSynchronize(s));
        loc.release();
        g.n = n;
        g.m = mloc;
        g.w_f64 = weights_f64 ? 1 : 0;
        slpa_graph_validate(ctx, g.base, g.w_f64);
        mark_partitioned(ctx, v_begin, v_end);
    });
}

int32_t slpa_part_gen_rmat(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB, uint32_t tABC,
                           uint64_t seed, int32_t permute, uint64_t perm_key, int64_t v_begin, int64_t v_end) {
    return guard(ctx, [&] {
        slpa_part_gen_rmat_impl(ctx, scale, num_edges, tA, tAB, tABC, seed, permute, perm_key, v_begin, v_end);
        mark_partitioned(ctx, v_begin, v_end);
    });
}

int32_t slpa_rmat_cuts(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB, uint32_t tABC,
                       uint64_t seed, int32_t permute, uint64_t perm_key, int32_t world, int64_t *cuts) {
    return guard(ctx, [&] {
        SLPA_REQUIRE(cuts != nullptr, SLPA_EINVAL, "cuts is NULL");
        slpa_rmat_cuts_impl(ctx, scale, num_edges, tA, tAB, tABC, seed, permute, perm_key, world, cuts);
    });
}

int32_t slpa_part_arc_hash(slpa_ctx *ctx, uint64_t *hash4) {
    return guard(ctx, [&] {
        require_part(ctx);
        SLPA_REQUIRE(hash4 != nullptr, SLPA_EINVAL, "hash4 is NULL");
        slpa_arc_hash_impl(ctx, hash4);
    });
}

int32_t slpa_part_set_symmetric(slpa_ctx *ctx, int32_t symmetric) {
    return guard(ctx, [&] {
        require_part(ctx);
        ctx->g.symmetric = symmetric ? 1 : 0;
        ctx->part_sym_known = 1;
    });
}

int32_t slpa_part_info(slpa_ctx *ctx, int64_t *n, int64_t *m_local, int64_t *v_begin, int64_t *v_end) {
    return guard(ctx, [&] {
        require_part(ctx);
        *n = ctx->g.n;
        *m_local = ctx->g.m;
        *v_begin = ctx->v_begin;
        *v_end = ctx->v_end;
    });
}

int32_t slpa_part_buffers(slpa_ctx *ctx, uint64_t *labels_dptr, uint64_t *flags_dptr) {
    return guard(ctx, [&] {
        require_part(ctx);
        SLPA_REQUIRE(ctx->wb.lab_old.p && ctx->wb.flag_a.p, SLPA_EINVAL, "call slpa_part_begin first");
        *labels_dptr = (uint64_t)(uintptr_t)ctx->wb.lab_old.p;
        *flags_dptr = (uint64_t)(uintptr_t)ctx->wb.flag_a.p;
    });
}

// Start a partitioned lpa_run: labels = arange(n) (lpa.py:289), owned
// vertices unprocessed (lpa.py:290), no outgoing marks.  worker_count > 0:
// asynchronous sweeps (slpa_part_sweep); worker_count == 0: deterministic
// sweeps driven round by round (slpa_part_det_round / _import / _commit).
int32_t slpa_part_begin(slpa_ctx *ctx, const slpa_config *cfg) {
    return guard(ctx, [&] {
        slpa_validate_config(cfg);
        require_part(ctx);
        slpa_ensure_bins(ctx, cfg);
        slpa_alloc_work(ctx);
        if (cfg->worker_count == 0) ctx->wb.dirty_bytes.alloc((size_t)ctx->g.n);
        ctx->stats = slpa_run_stats{};
        slpa_init_labels(ctx);
        const int64_t n = ctx->g.n;
        if (ctx->v_begin > 0) CUDA_TRY(cudaMemsetAsync(ctx->wb.flag_a.p, 0, (size_t)ctx->v_begin, ctx->stream));
        if (ctx->v_end < n)
            CUDA_TRY(cudaMemsetAsync(ctx->wb.flag_a.p + ctx->v_end, 0, (size_t)(n - ctx->v_end), ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        ctx->have_labels = 1;
    });
}

int32_t slpa_part_sweep(slpa_ctx *ctx, const slpa_config *cfg, int32_t pickless, int64_t *changed_local) {
    return guard(ctx, [&] {
        slpa_validate_config(cfg);
        require_part(ctx);
        slpa_ensure_bins(ctx, cfg);
        *changed_local = slpa_sweep_async(ctx, cfg, pickless ? 1 : 0);
        ctx->stats.sweeps += 1;
    });
}

int32_t slpa_part_det_buffers(slpa_ctx *ctx, uint64_t *lab_new_dptr, uint64_t *dirty_bytes_dptr) {
    return guard(ctx, [&] {
        require_part(ctx);
        SLPA_REQUIRE(ctx->wb.lab_new.p && ctx->wb.dirty_bytes.p, SLPA_EINVAL,
                     "call slpa_part_begin with worker_count == 0 first");
        *lab_new_dptr = (uint64_t)(uintptr_t)ctx->wb.lab_new.p;
        *dirty_bytes_dptr = (uint64_t)(uintptr_t)ctx->wb.dirty_bytes.p;
    });
}

int32_t slpa_part_det_round(slpa_ctx *ctx, const slpa_config *cfg, int32_t pickless, int32_t round) {
    return guard(ctx, [&] {
        slpa_validate_config(cfg);
        require_part(ctx);
        SLPA_REQUIRE(cfg->worker_count == 0, SLPA_EINVAL, "deterministic rounds need worker_count == 0");
        SLPA_REQUIRE(ctx->part_sym_known && ctx->g.symmetric, SLPA_EUNSUPPORTED,
                     "partitioned deterministic sweeps need a symmetric graph (confirmed with "
                     "slpa_part_arc_hash / slpa_part_set_symmetric)");
        SLPA_REQUIRE(ctx->wb.dirty_bytes.p, SLPA_EINVAL, "call slpa_part_begin with worker_count == 0 first");
        slpa_ensure_bins(ctx, cfg);
        slpa_part_det_round_impl(ctx, cfg, pickless ? 1 : 0, round);
    });
}

int32_t slpa_part_det_import(slpa_ctx *ctx, int64_t *dirty_total) {
    return guard(ctx, [&] {
        require_part(ctx);
        SLPA_REQUIRE(ctx->wb.dirty_bytes.p, SLPA_EINVAL, "call slpa_part_begin with worker_count == 0 first");
        *dirty_total = slpa_part_det_import_impl(ctx);
    });
}

int32_t slpa_part_det_commit(slpa_ctx *ctx, const slpa_config *cfg, int64_t *changed_local) {
    return guard(ctx, [&] {
        slpa_validate_config(cfg);
        require_part(ctx);
        SLPA_REQUIRE(ctx->wb.dirty_bytes.p, SLPA_EINVAL, "call slpa_part_begin with worker_count == 0 first");
        *changed_local = slpa_part_det_commit_impl(ctx, cfg);
    });
}

int32_t slpa_part_end_exchange(slpa_ctx *ctx) {
    return guard(ctx, [&] {
        require_part(ctx);
        const int64_t n = ctx->g.n;
        if (ctx->v_begin > 0) CUDA_TRY(cudaMemsetAsync(ctx->wb.flag_a.p, 0, (size_t)ctx->v_begin, ctx->stream));
        if (ctx->v_end < n)
            CUDA_TRY(cudaMemsetAsync(ctx->wb.flag_a.p + ctx->v_end, 0, (size_t)(n - ctx->v_end), ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    });
}

int32_t slpa_part_tally(slpa_ctx *ctx, double *internal_local, uint64_t *incident_dptr, uint64_t *sizes_dptr) {
    return guard(ctx, [&] {
        require_part(ctx);
        SLPA_REQUIRE(ctx->have_labels, SLPA_EINVAL, "no labels resident");
        slpa_part_tally_impl(ctx, internal_local, incident_dptr, sizes_dptr);
    });
}

int32_t slpa_part_modularity(slpa_ctx *ctx, double internal_total, double *q) {
    return guard(ctx, [&] {
        require_part(ctx);
        slpa_part_modularity_impl(ctx, internal_total, q);
    });
}

}  // extern "C"
