// slpa_api.cu -- the extern "C" boundary (include/slpa.h) and the host-side
// outer loop of lpa_run (lpa.py:262-308).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <vector>
#include "slpa_internal.cuh"

void slpa_graph_validate(slpa_ctx *ctx, const Csr &c, int w_f64);
void slpa_gen_rmat_impl(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB, uint32_t tABC,
                        uint64_t seed, int32_t permute, uint64_t perm_key);
void slpa_gen_grid_impl(slpa_ctx *ctx, int64_t rows, int64_t cols, int32_t permute, uint64_t perm_key);
void slpa_gen_kmer_impl(slpa_ctx *ctx, int64_t n, uint32_t keep, uint64_t seed, int32_t permute, uint64_t perm_key);
void slpa_build_graph_impl(slpa_ctx *ctx, int64_t n, int64_t ne, const int64_t *src, const int64_t *dst,
                           const double *w, int32_t weights_f64);
void slpa_validate_graph_impl(slpa_ctx *ctx, int32_t *code, int64_t *vertex, double *deg_sum, double *total);

namespace {
thread_local std::string g_create_err;

template <class F>
int32_t guard(slpa_ctx *ctx, F &&f) {
    try {
        if (ctx) {
            ctx->err.clear();
            cudaError_t e = cudaSetDevice(ctx->device);
            if (e != cudaSuccess) throw SlpaError{SLPA_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)};
        }
        f();
        return SLPA_OK;
    } catch (const SlpaError &e) {
        if (ctx) ctx->err = e.msg;
        else g_create_err = e.msg;
        return e.code;
    } catch (const std::exception &e) {
        if (ctx) ctx->err = e.what();
        else g_create_err = e.what();
        return SLPA_ECUDA;
    }
}

void require_graph(slpa_ctx *ctx) { SLPA_REQUIRE(ctx->g.base.off.p != nullptr, SLPA_ENOGRAPH, "no graph uploaded"); }

void upload_csr(slpa_ctx *ctx, int64_t n, int64_t m, const int64_t *off, const int32_t *tgt, const void *w,
                int32_t w_f64, cudaMemcpyKind kind) {
    SLPA_REQUIRE(n >= 0 && m >= 0, SLPA_EINVAL, "negative size");
    SLPA_REQUIRE(n < (1LL << 31) - 1, SLPA_EUNSUPPORTED, "more than 2^31-2 vertices");
    DeviceGraph &g = ctx->g;
    cudaStream_t s = ctx->stream;
    g.perm.release();
    g.ids.release();
    g.pos.release();
    g.has_order = 0;
    // buffers are reused when large enough (repeated lpa_run calls re-upload
    // the graph; freeing and re-allocating GBs would dominate)
    g.base.n = n;
    g.base.m = m;
    g.base.off.alloc(n + 1);
    g.base.tgt.alloc(m);
    CUDA_TRY(cudaMemcpyAsync(g.base.off.p, off, (n + 1) * sizeof(int64_t), kind, s));
    if (m) CUDA_TRY(cudaMemcpyAsync(g.base.tgt.p, tgt, m * sizeof(int32_t), kind, s));
    if (w_f64) {
        g.base.w32.release();
        g.base.w64.alloc(m);
        if (m) CUDA_TRY(cudaMemcpyAsync(g.base.w64.p, w, m * sizeof(double), kind, s));
    } else {
        g.base.w64.release();
        g.base.w32.alloc(m);
        if (m) CUDA_TRY(cudaMemcpyAsync(g.base.w32.p, w, m * sizeof(float), kind, s));
    }
    g.n = n;
    g.m = m;
    g.w_f64 = w_f64 ? 1 : 0;
    slpa_graph_validate(ctx, g.base, g.w_f64);
    ctx->have_labels = 0;
    ctx->part = 0;
}
}  // namespace

void slpa_validate_config(const slpa_config *cfg) {  // LpaConfig.validate (lpa.py:62-80)
    SLPA_REQUIRE(cfg != nullptr, SLPA_EINVAL, "config is NULL");
    SLPA_REQUIRE(cfg->variant >= 0 && cfg->variant <= 2, SLPA_EINVAL, "variant must be one of ('exact', 'bm', 'mg')");
    SLPA_REQUIRE(cfg->scan_mode == 0 || cfg->scan_mode == 1, SLPA_EINVAL,
                 "scan_mode must be one of ('single', 'double')");
    SLPA_REQUIRE(cfg->sketch_slots >= 1, SLPA_EINVAL, "sketch_slots must be at least 1");
    SLPA_REQUIRE(cfg->pickless_gap >= 1, SLPA_EINVAL, "pickless_gap must be at least 1");
    SLPA_REQUIRE(cfg->tolerance > 0 && cfg->tolerance <= 1, SLPA_EINVAL, "tolerance must be in (0, 1]");
    SLPA_REQUIRE(cfg->max_iterations >= 1, SLPA_EINVAL, "max_iterations must be at least 1");
    SLPA_REQUIRE(cfg->degree_threshold >= 1, SLPA_EINVAL, "degree_threshold must be at least 1");
    SLPA_REQUIRE(cfg->partial_groups >= 1, SLPA_EINVAL, "partial_groups must be at least 1");
    SLPA_REQUIRE(cfg->worker_count >= 0, SLPA_EINVAL, "worker_count must be non-negative");
}

void set_label_l2_window(slpa_ctx *ctx);

void slpa_alloc_work(slpa_ctx *ctx) {
    const int64_t n = ctx->g.n;
    WorkBuffers &wb = ctx->wb;
    wb.lab_old.alloc(n);
    wb.lab_new.alloc(n);
    wb.flag_a.alloc(n);
    wb.flag_b.alloc(n);
    wb.dirty_a.alloc(n / 32 + 1);
    wb.dirty_b.alloc(n / 32 + 1);
    if (ctx->g.n_giant > 0) {
        wb.dirty_g.alloc(n / 32 + 1);
        wb.dirty_gp.alloc(n / 32 + 1);
    }
    wb.wl_lo.alloc(n);  // (bins are filled before the work buffers: the worklists are sized by class)
    wb.wl_mid.alloc(ctx->g.n_mid + 1);
    wb.wl_hi.alloc(ctx->g.n_hi + 1);
    wb.wl_giant.alloc(ctx->g.n_giant + 1);
    wb.glab.alloc(ctx->g.giant_arcs + 1);
    wb.gw.alloc((ctx->g.giant_arcs + 1) * (ctx->g.w_f64 ? sizeof(double) : sizeof(float)));
    wb.io_labels.alloc(n);
    wb.io_flags.alloc(n);
    wb.counters.alloc(CNT_TOTAL);
    if (ctx->prof_on) wb.tbits.alloc(n / 32 + 1);
    wb.fbits.alloc(n / 32 + 1);
    CUDA_TRY(cudaMemsetAsync(wb.dirty_a.p, 0, (n / 32 + 1) * sizeof(uint32_t), ctx->stream));
    CUDA_TRY(cudaMemsetAsync(wb.dirty_b.p, 0, (n / 32 + 1) * sizeof(uint32_t), ctx->stream));
    if (!ctx->h_counters) CUDA_TRY(cudaMallocHost((void **)&ctx->h_counters, CNT_TOTAL * sizeof(unsigned long long)));
    set_label_l2_window(ctx);
}

// Keep the label array the sweeps gather from (lab_new, 4 B per vertex) in
// L2: an access-policy window on both streams marks it persisting, so the
// streamed CSR (loaded evict-first) does not push it out.  SLPA_L2_PERSIST_MB
// caps the set-aside (default: the device maximum, 79 MiB on the B200, which
// covers the 64 MiB label words of RMAT s24; 0 disables).  The process-wide
// limit in force before the first window is saved and restored, and the
// persisting lines are reset, at the end of every run and in slpa_destroy
// (release_label_l2_window) so other work in the process gets its L2 back.
void set_label_l2_window(slpa_ctx *ctx) {
    static const long cap_mb = [] {
        const char *e = getenv("SLPA_L2_PERSIST_MB");
        return e ? atol(e) : 4096L;
    }();
    if (cap_mb <= 0 || ctx->g.n == 0) return;
    int max_persist = 0, max_window = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device));
    CUDA_TRY(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device));
    const size_t want = (size_t)ctx->g.n * sizeof(uint32_t);
    const size_t setaside = std::min<size_t>(std::min<size_t>((size_t)max_persist, (size_t)cap_mb << 20),
                                             (want + (1u << 20) - 1) & ~(size_t)((1u << 20) - 1));
    if (setaside == 0 || max_window <= 0) return;
    if (!ctx->l2_saved) {
        CUDA_TRY(cudaDeviceGetLimit(&ctx->l2_prev_limit, cudaLimitPersistingL2CacheSize));
        ctx->l2_saved = 1;
    }
    CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside));
    cudaStreamAttrValue attr{};
    attr.accessPolicyWindow.base_ptr = ctx->wb.lab_new.p;
    attr.accessPolicyWindow.num_bytes = std::min<size_t>(want, (size_t)max_window);
    attr.accessPolicyWindow.hitRatio = std::min(1.0f, (float)setaside / (float)attr.accessPolicyWindow.num_bytes);
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CUDA_TRY(cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &attr));
    if (ctx->stream2) CUDA_TRY(cudaStreamSetAttribute(ctx->stream2, cudaStreamAttributeAccessPolicyWindow, &attr));
    if (getenv("SLPA_TRACE"))
        fprintf(stderr, "[slpa] L2 persisting window: %zu bytes of %zu, set-aside %zu (max %d, window max %d)\n",
                (size_t)attr.accessPolicyWindow.num_bytes, want, setaside, max_persist, max_window);
}

// Undo set_label_l2_window: clear the stream windows, demote the persisting
// lines to normal and restore the process's previous set-aside.
void release_label_l2_window(slpa_ctx *ctx) {
    if (!ctx->l2_saved) return;
    cudaStreamAttrValue attr{};
    attr.accessPolicyWindow.num_bytes = 0;
    if (ctx->stream) cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
    if (ctx->stream2) cudaStreamSetAttribute(ctx->stream2, cudaStreamAttributeAccessPolicyWindow, &attr);
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, ctx->l2_prev_limit);
    ctx->l2_saved = 0;
}

static void reset_stats(slpa_ctx *ctx) {
    ctx->stats = slpa_run_stats{};
}

static void fill_mem_stats(slpa_ctx *ctx) {
    ctx->stats.device_bytes = (int64_t)(ctx->g.bytes() + ctx->wb.bytes());
    ctx->stats.graph_bytes = (int64_t)ctx->g.csr_bytes();
}

extern "C" {

const char *slpa_version(void) { return "slpa_b200 0.1.0 (sm_100a)"; }

int32_t slpa_create(int32_t device, slpa_ctx **out) {
    return guard(nullptr, [&] {
        SLPA_REQUIRE(out != nullptr, SLPA_EINVAL, "out is NULL");
        int count = 0;
        CUDA_TRY(cudaGetDeviceCount(&count));
        SLPA_REQUIRE(device >= 0 && device < count, SLPA_EINVAL, "no such CUDA device");
        CUDA_TRY(cudaSetDevice(device));
        cudaDeviceProp prop;
        CUDA_TRY(cudaGetDeviceProperties(&prop, device));
        SLPA_REQUIRE(prop.major == 10, SLPA_EUNSUPPORTED,
                     std::string("libslpa_b200 is built for sm_100a (B200); device is ") + prop.name);
        slpa_ctx *c = new slpa_ctx();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        try {
            CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            CUDA_TRY(cudaEventCreate(&c->ev0));
            CUDA_TRY(cudaEventCreate(&c->ev1));
            CUDA_TRY(cudaEventCreate(&c->pev0));
            CUDA_TRY(cudaEventCreate(&c->pev1));
            // giants run on a higher-priority stream: their long sequential
            // chunk chains must start as soon as SMs free up, not after the
            // concurrent high-degree scan has drained
            int prio_lo = 0, prio_hi = 0;
            CUDA_TRY(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
            CUDA_TRY(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, prio_hi));
            CUDA_TRY(cudaEventCreateWithFlags(&c->gev0, cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&c->gev1, cudaEventDisableTiming));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int32_t slpa_destroy(slpa_ctx *ctx) {
    if (!ctx) return SLPA_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    release_label_l2_window(ctx);
    ctx->g.base.release();
    ctx->g.perm.release();
    ctx->g.ids.release();
    ctx->g.pos.release();
    ctx->g.roff.release();
    ctx->g.rsrc.release();
    ctx->g.cls.release();
    ctx->g.bin_lo.release();
    ctx->g.bin_mid.release();
    ctx->g.bin_hi.release();
    ctx->g.bin_giant.release();
    ctx->g.giant_off.release();
    ctx->g.sort_k1.release();
    ctx->g.sort_k2.release();
    ctx->g.sort_small.release();
    ctx->g.sort_v.release();
    WorkBuffers &wb = ctx->wb;
    wb.lab_old.release(); wb.lab_new.release(); wb.flag_a.release(); wb.flag_b.release();
    wb.dirty_a.release(); wb.dirty_b.release(); wb.wl_lo.release(); wb.wl_mid.release(); wb.wl_hi.release(); wb.wl_giant.release();
    wb.glab.release(); wb.gw.release();
    wb.io_labels.release(); wb.io_flags.release(); wb.counters.release(); wb.metric_d.release();
    wb.metric_u.release(); wb.scratch.release();
    wb.hparts.release(); wb.hmeta.release(); wb.dirty_g.release(); wb.dirty_gp.release();
    wb.dirty_bytes.release(); wb.dcount.release(); wb.tbits.release(); wb.fbits.release(); wb.xscratch.release();
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    ctx->h_stage = nullptr;
    ctx->h_stage_n = 0;
    if (ctx->h_counters) cudaFreeHost(ctx->h_counters);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->pev0) cudaEventDestroy(ctx->pev0);
    if (ctx->pev1) cudaEventDestroy(ctx->pev1);
    if (ctx->gev0) cudaEventDestroy(ctx->gev0);
    if (ctx->gev1) cudaEventDestroy(ctx->gev1);
    if (ctx->stream2) {
        cudaStreamSynchronize(ctx->stream2);
        cudaStreamDestroy(ctx->stream2);
    }
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return SLPA_OK;
}

const char *slpa_last_error(const slpa_ctx *ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int32_t slpa_stream(slpa_ctx *ctx, uint64_t *stream_out) {
    return guard(ctx, [&] { *stream_out = (uint64_t)(uintptr_t)ctx->stream; });
}

int32_t slpa_graph_upload(slpa_ctx *ctx, int64_t n, int64_t m, const int64_t *offsets, const int32_t *targets,
                          const void *weights, int32_t weights_f64, const int64_t *order) {
    return guard(ctx, [&] {
        upload_csr(ctx, n, m, offsets, targets, weights, weights_f64, cudaMemcpyHostToDevice);
        slpa_graph_apply_order(ctx, order, false);
    });
}

int32_t slpa_graph_upload_device(slpa_ctx *ctx, int64_t n, int64_t m, const int64_t *offsets, const int32_t *targets,
                                 const void *weights, int32_t weights_f64, const int64_t *order) {
    return guard(ctx, [&] {
        upload_csr(ctx, n, m, offsets, targets, weights, weights_f64, cudaMemcpyDeviceToDevice);
        slpa_graph_apply_order(ctx, order, true);
    });
}

int32_t slpa_graph_set_order(slpa_ctx *ctx, const int64_t *order) {
    return guard(ctx, [&] {
        require_graph(ctx);
        slpa_graph_apply_order(ctx, order, false);
        ctx->have_labels = 0;
    });
}

int32_t slpa_graph_info(slpa_ctx *ctx, int64_t *n, int64_t *m, int32_t *weights_f64, int32_t *symmetric) {
    return guard(ctx, [&] {
        require_graph(ctx);
        if (n) *n = ctx->g.n;
        if (m) *m = ctx->g.m;
        if (weights_f64) *weights_f64 = ctx->g.w_f64;
        if (symmetric) *symmetric = ctx->g.symmetric;
    });
}

int32_t slpa_graph_download(slpa_ctx *ctx, int64_t *offsets, int32_t *targets, void *weights) {
    return guard(ctx, [&] {
        require_graph(ctx);
        const Csr &c = ctx->g.base;
        cudaStream_t s = ctx->stream;
        if (offsets) CUDA_TRY(cudaMemcpyAsync(offsets, c.off.p, (c.n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        if (targets && c.m) CUDA_TRY(cudaMemcpyAsync(targets, c.tgt.p, c.m * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        if (weights && c.m) {
            if (ctx->g.w_f64)
                CUDA_TRY(cudaMemcpyAsync(weights, c.w64.p, c.m * sizeof(double), cudaMemcpyDeviceToHost, s));
            else
                CUDA_TRY(cudaMemcpyAsync(weights, c.w32.p, c.m * sizeof(float), cudaMemcpyDeviceToHost, s));
        }
        CUDA_TRY(cudaStreamSynchronize(s));
    });
}

int32_t slpa_gen_rmat(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB, uint32_t tABC,
                      uint64_t seed, int32_t permute, uint64_t perm_key) {
    return guard(ctx, [&] {
        ctx->part = 0;
        slpa_gen_rmat_impl(ctx, scale, num_edges, tA, tAB, tABC, seed, permute, perm_key);
        slpa_graph_finalize(ctx);
        ctx->have_labels = 0;
    });
}

int32_t slpa_gen_grid(slpa_ctx *ctx, int64_t rows, int64_t cols, int32_t permute, uint64_t perm_key) {
    return guard(ctx, [&] {
        ctx->part = 0;
        slpa_gen_grid_impl(ctx, rows, cols, permute, perm_key);
        slpa_graph_finalize(ctx);
        ctx->have_labels = 0;
    });
}

int32_t slpa_gen_kmer(slpa_ctx *ctx, int64_t n, uint32_t keep, uint64_t seed, int32_t permute, uint64_t perm_key) {
    return guard(ctx, [&] {
        ctx->part = 0;
        slpa_gen_kmer_impl(ctx, n, keep, seed, permute, perm_key);
        slpa_graph_finalize(ctx);
        ctx->have_labels = 0;
    });
}

int32_t slpa_build_graph(slpa_ctx *ctx, int64_t n, int64_t num_edges, const int64_t *src, const int64_t *dst,
                         const double *w, int32_t weights_f64) {
    return guard(ctx, [&] {
        ctx->part = 0;
        slpa_build_graph_impl(ctx, n, num_edges, src, dst, w, weights_f64);
        slpa_graph_finalize(ctx);
        ctx->have_labels = 0;
    });
}

int32_t slpa_validate_graph(slpa_ctx *ctx, int32_t *code, int64_t *vertex, double *deg_sum, double *total) {
    return guard(ctx, [&] {
        require_graph(ctx);
        slpa_validate_graph_impl(ctx, code, vertex, deg_sum, total);
    });
}

int32_t slpa_run(slpa_ctx *ctx, const slpa_config *cfg, int32_t *labels_out, int64_t *delta_history,
                 int32_t *iterations, int32_t *converged, slpa_hook_fn hook, void *hook_user) {
    return guard(ctx, [&] {
        slpa_validate_config(cfg);
        require_graph(ctx);
        SLPA_REQUIRE(delta_history && iterations && converged, SLPA_EINVAL, "output pointers are NULL");
        DeviceGraph &g = ctx->g;
        const auto tp0 = std::chrono::steady_clock::now();
        slpa_ensure_bins(ctx, cfg);
        slpa_alloc_work(ctx);
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        const auto tp1 = std::chrono::steady_clock::now();
        reset_stats(ctx);
        ctx->have_labels = 0;
        const bool det = cfg->worker_count == 0;
        const int64_t n = g.n;
        // The hook gets the live labels (lpa.py:271-273): the caller's output
        // buffer when given; an edit it makes is uploaded before the next sweep.
        std::vector<int32_t> hook_buf, hook_prev;
        int32_t *hb = labels_out;
        if (hook) {
            if (!hb) {
                hook_buf.resize((size_t)std::max<int64_t>(n, 1));
                hb = hook_buf.data();
            }
            hook_prev.resize((size_t)std::max<int64_t>(n, 1));
        }
        CUDA_TRY(cudaEventRecord(ctx->ev0, ctx->stream));
        slpa_init_labels(ctx);
        int32_t it = 0, conv = 0;
        for (; it < cfg->max_iterations;) {
            const int pickless = (it % cfg->pickless_gap) == 0;  // lpa.py:294
            const int64_t delta = n ? (det ? slpa_sweep_det(ctx, cfg, pickless) : slpa_sweep_async(ctx, cfg, pickless)) : 0;
            delta_history[it] = delta;
            ctx->stats.sweeps += 1;
            ++it;
            if (hook) {  // lpa.py:297-298
                slpa_labels_to_host(ctx, hb);
                if (n) std::memcpy(hook_prev.data(), hb, (size_t)n * sizeof(int32_t));
                if (hook(hook_user, it - 1, pickless, hb) != 0)
                    throw SlpaError{SLPA_EHOOK, "iteration hook raised"};
                if (n && std::memcmp(hook_prev.data(), hb, (size_t)n * sizeof(int32_t)) != 0) {
                    if (cfg->variant == SLPA_VARIANT_EXACT)
                        for (int64_t i = 0; i < n; ++i)
                            SLPA_REQUIRE(hb[i] >= 0, SLPA_EINVAL, "'list' argument must have no negative elements");
                    slpa_labels_from_host(ctx, hb);  // the edited live array feeds the next sweep
                }
            }
            const double frac = n ? (double)delta / (double)n : 0.0;  // lpa.py:299
            if (!pickless && frac < cfg->tolerance) {
                conv = 1;
                break;
            }
        }
        CUDA_TRY(cudaEventRecord(ctx->ev1, ctx->stream));
        CUDA_TRY(cudaEventSynchronize(ctx->ev1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->stats.device_ms = ms;
        fill_mem_stats(ctx);
        *iterations = it;
        *converged = conv;
        ctx->have_labels = 1;
        release_label_l2_window(ctx);
        const auto tp2 = std::chrono::steady_clock::now();
        if (labels_out) slpa_labels_to_host(ctx, labels_out);
        if (getenv("SLPA_TRACE")) {
            const auto tp3 = std::chrono::steady_clock::now();
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            fprintf(stderr, "[slpa] run phases: bins+alloc %.2f ms, sweeps %.2f ms (device %.2f), labels D2H %.2f ms\n",
                    ms(tp0, tp1), ms(tp1, tp2), (double)ctx->stats.device_ms, ms(tp2, tp3));
        }
    });
}

int32_t slpa_move(slpa_ctx *ctx, const slpa_config *cfg, int32_t *labels, uint8_t *unprocessed, int32_t pickless,
                  int64_t *changed) {
    return guard(ctx, [&] {
        slpa_validate_config(cfg);
        require_graph(ctx);
        SLPA_REQUIRE(labels && unprocessed && changed, SLPA_EINVAL, "NULL argument");
        const int64_t n = ctx->g.n;
        if (cfg->variant == SLPA_VARIANT_EXACT)  // np.bincount rejects negative labels (lpa.py:104)
            for (int64_t i = 0; i < n; ++i)
                SLPA_REQUIRE(labels[i] >= 0, SLPA_EINVAL, "'list' argument must have no negative elements");
        slpa_ensure_bins(ctx, cfg);
        slpa_alloc_work(ctx);
        reset_stats(ctx);
        if (n == 0) {
            *changed = 0;
            return;
        }
        slpa_labels_from_host(ctx, labels);
        slpa_flags_from_host(ctx, unprocessed);
        const int64_t delta =
            cfg->worker_count == 0 ? slpa_sweep_det(ctx, cfg, pickless ? 1 : 0) : slpa_sweep_async(ctx, cfg, pickless ? 1 : 0);
        ctx->stats.sweeps = 1;
        slpa_labels_to_host(ctx, labels);
        slpa_flags_to_host(ctx, unprocessed);
        *changed = delta;
        ctx->have_labels = 1;
        fill_mem_stats(ctx);
    });
}

int32_t slpa_get_labels(slpa_ctx *ctx, int32_t *labels_out) {
    return guard(ctx, [&] {
        SLPA_REQUIRE(ctx->have_labels, SLPA_EINVAL, "no labels resident (run first)");
        slpa_labels_to_host(ctx, labels_out);
    });
}

int32_t slpa_set_profiling(slpa_ctx *ctx, int32_t on) {
    return guard(ctx, [&] {
        ctx->prof_on = on ? 1 : 0;
        ctx->prof = slpa_profile{};
    });
}

int32_t slpa_get_profile(slpa_ctx *ctx, slpa_profile *out) {
    return guard(ctx, [&] { *out = ctx->prof; });
}

int32_t slpa_last_run_stats(slpa_ctx *ctx, slpa_run_stats *out) {
    return guard(ctx, [&] { *out = ctx->stats; });
}

int64_t slpa_aux_memory_estimate(int64_t n, int32_t value_bytes, const slpa_config *cfg) {  // lpa.py:311-333
    const int64_t workers = std::max<int64_t>(cfg->worker_count, 1);
    const int64_t base = n * (4 + 1);
    int64_t per;
    if (cfg->variant == SLPA_VARIANT_EXACT) per = n * (4 + value_bytes);
    else if (cfg->variant == SLPA_VARIANT_MG) per = (int64_t)cfg->partial_groups * cfg->sketch_slots * (4 + value_bytes);
    else per = (int64_t)cfg->partial_groups * (4 + value_bytes);
    return base + workers * per;
}

int32_t slpa_modularity(slpa_ctx *ctx, const int32_t *labels, double *q, int64_t *num_communities, int64_t *sizes,
                        double *internal, double *incident) {
    return guard(ctx, [&] {
        require_graph(ctx);
        const int64_t n = ctx->g.n;
        ctx->wb.io_labels.alloc(n);
        ctx->wb.lab_old.alloc(n);
        const int32_t *d_lab;
        if (labels) {
            // labels by vertex id -> by position
            if (ctx->g.has_order) {
                DevBuf<int32_t> tmp;
                tmp.alloc(n);
                CUDA_TRY(cudaMemcpyAsync(tmp.p, labels, n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
                slpa_permute_id_to_pos(ctx, tmp.p, ctx->wb.io_labels.p);  // io[p] = labels[ids[p]]
                CUDA_TRY(cudaStreamSynchronize(ctx->stream));
                tmp.release();
            } else {
                CUDA_TRY(cudaMemcpyAsync(ctx->wb.io_labels.p, labels, n * sizeof(int32_t), cudaMemcpyHostToDevice,
                                         ctx->stream));
            }
            d_lab = ctx->wb.io_labels.p;
        } else {
            SLPA_REQUIRE(ctx->have_labels, SLPA_EINVAL, "no labels resident (run first)");
            d_lab = ctx->wb.lab_old.p;
        }
        slpa_tally(ctx, d_lab, q, num_communities, sizes, internal, incident);
    });
}

}  // extern "C"
