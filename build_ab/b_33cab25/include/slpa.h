/*
 * slpa.h -- C ABI of the B200-native label-propagation engine
 *           (libslpa_b200.so, built from paper_2411_19901_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's hot path
 * (sketchlpa 0.1.0, /root/reference/pkg/src/sketchlpa).  Each entry point
 * names the reference interface it replaces.  Plain C types only: host
 * pointers unless a name says `_device`.  Every call returns an slpa_status;
 * slpa_last_error() gives the message.  A context owns one device, one
 * stream, one resident graph and its work buffers; contexts are independent
 * (no hidden globals), so one context per device / per thread.
 */
#ifndef SLPA_H
#define SLPA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SLPA_OK = 0,
    SLPA_EINVAL = 1,      /* bad argument / config  -> ValueError (lpa.py:62-80, :287-288; metrics.py:36-40, :71-72) */
    SLPA_ECUDA = 2,       /* CUDA runtime failure   -> RuntimeError */
    SLPA_EUNSUPPORTED = 3,/* option outside the GPU path's limits -> ValueError */
    SLPA_ENOGRAPH = 4,    /* no graph resident */
    SLPA_EHOOK = 5        /* iteration hook asked to abort (exception in the Python hook) */
} slpa_status;

enum { SLPA_VARIANT_EXACT = 0, SLPA_VARIANT_BM = 1, SLPA_VARIANT_MG = 2 };
enum { SLPA_SCAN_SINGLE = 0, SLPA_SCAN_DOUBLE = 1 };

/* Mirror of LpaConfig (lpa.py:44-60); validated like LpaConfig.validate()
 * (lpa.py:62-80).  worker_count == 0 selects the deterministic mode whose
 * results are bit-identical to the reference's sequential sweep
 * (lpa.py:204-224); worker_count > 0 selects the asynchronous in-place GPU
 * sweep (the analogue of the reference's threaded mode, lpa.py:242-259). */
typedef struct {
    int32_t variant;          /* SLPA_VARIANT_*                 lpa.py:51 */
    int32_t scan_mode;        /* SLPA_SCAN_*                    lpa.py:52 */
    int32_t sketch_slots;     /* k                              lpa.py:53 */
    int32_t pickless_gap;     /* rho                            lpa.py:54 */
    double  tolerance;        /* tau                            lpa.py:55 */
    int32_t max_iterations;   /*                                lpa.py:56 */
    int32_t degree_threshold; /* D_H                            lpa.py:57 */
    int32_t partial_groups;   /* R_H                            lpa.py:58 */
    int32_t worker_count;     /* 0 = deterministic, >0 = async  lpa.py:59 */
    int32_t shared_sketch;    /*                                lpa.py:60 */
} slpa_config;

/* Called after every sweep, like iteration_hook(it, pickless, labels)
 * (lpa.py:271-273, :297-298).  `labels` is a host copy indexed by vertex id.
 * Return non-zero to abort the run (slpa_run then returns SLPA_EHOOK). */
typedef int32_t (*slpa_hook_fn)(void *user, int32_t iteration, int32_t pickless, const int32_t *labels);

typedef struct slpa_ctx slpa_ctx;

/* Per-run counters (not part of the reference API; for measurement). */
typedef struct {
    int64_t sweeps;             /* iterations executed */
    int64_t rounds;             /* speculative rounds (deterministic mode) */
    int64_t vertex_evals;       /* vertex evaluations incl. re-evaluations */
    int64_t arc_reads;          /* adjacency arcs scanned incl. re-evaluations */
    int64_t first_evals;        /* vertices the sequential sweep processes (turn taken), summed over sweeps;
                                   deterministic mode: profiling runs only (0 otherwise) */
    int64_t first_arcs;         /* arcs of those vertices (the algorithmic arcs) */
    double  device_ms;          /* device time of the last run (CUDA events) */
    int64_t device_bytes;       /* bytes the context holds on the device */
    int64_t graph_bytes;        /* of which the resident CSR */
    int64_t kernel_launches;    /* kernels launched by the last run / move */
} slpa_run_stats;

/* Per-kernel-class device time when profiling is on (CUDA events on the
 * context stream around every launch; adds a host sync per launch, so keep
 * it off for throughput runs).  evals / arcs are the vertices evaluated and
 * arcs scanned by those launches -- the algorithmic work. */
enum {
    SLPA_PROF_EVAL_LO0 = 0,  /* round-0 label scan, deg < D_H (lane per vertex) */
    SLPA_PROF_EVAL_MID0 = 1, /* round-0 label scan, D_H <= deg < split (lane per vertex, R_H chunks) */
    SLPA_PROF_EVAL_HI0 = 2,  /* round-0 label scan, deg >= split (warp per vertex, lane = chunk) */
    SLPA_PROF_EVAL_LOK = 3,  /* re-evaluation rounds, same classes */
    SLPA_PROF_EVAL_MIDK = 4,
    SLPA_PROF_EVAL_HIK = 5,
    SLPA_PROF_COMPACT = 6,   /* dirty bitmap -> worklists */
    SLPA_PROF_COMMIT = 7,    /* label update, flags, changed-vertex count */
    SLPA_PROF_OTHER = 8,
    SLPA_PROF_EVAL_GIANT = 9,/* deg >= giant threshold: gather + warp-per-vertex replay (all rounds) */
    SLPA_PROF_N = 12
};
typedef struct {
    int64_t launches[SLPA_PROF_N];
    double ms[SLPA_PROF_N];
    int64_t evals[SLPA_PROF_N];
    int64_t arcs[SLPA_PROF_N];
} slpa_profile;

/* ---------------------------------------------------------------- context */
int32_t slpa_create(int32_t device, slpa_ctx **out);
int32_t slpa_destroy(slpa_ctx *ctx);
const char *slpa_last_error(const slpa_ctx *ctx);   /* ctx may be NULL (creation errors) */
const char *slpa_version(void);
/* The CUDA stream all work is issued on (cudaStream_t as an integer). */
int32_t slpa_stream(slpa_ctx *ctx, uint64_t *stream_out);

/* ------------------------------------------------------------ graph upload
 * Replaces handing a sketchlpa Graph (graph.py:35-74: offsets int64[n+1],
 * targets int32[m], weights float32|float64[m]) to lpa_run/lpa_move.  The
 * library copies the arrays (the caller's Graph stays immutable,
 * graph.py:73-74), checks the Graph invariants (graph.py:55-68), detects
 * whether the arc set is symmetric, and, when `order` is given (lpa.py:283-
 * 288, a permutation of 0..n-1), stores vertices in visiting order while
 * label values stay original ids. */
int32_t slpa_graph_upload(slpa_ctx *ctx, int64_t n, int64_t m, const int64_t *offsets,
                          const int32_t *targets, const void *weights, int32_t weights_f64,
                          const int64_t *order);
/* Same, from device pointers (e.g. torch CUDA tensors' data_ptr()). */
int32_t slpa_graph_upload_device(slpa_ctx *ctx, int64_t n, int64_t m, const int64_t *offsets,
                                 const int32_t *targets, const void *weights, int32_t weights_f64,
                                 const int64_t *order);
/* Re-order the resident graph for a new `order` (NULL = ascending ids). */
int32_t slpa_graph_set_order(slpa_ctx *ctx, const int64_t *order);
int32_t slpa_graph_info(slpa_ctx *ctx, int64_t *n, int64_t *m, int32_t *weights_f64, int32_t *symmetric);
/* Copy the resident CSR (in original id order) back to host buffers. */
int32_t slpa_graph_download(slpa_ctx *ctx, int64_t *offsets, int32_t *targets, void *weights);

/* ----------------------------------------------------- synthetic graphs
 * Device-side generators + canonical assembly (graph.py:107-139 rules:
 * unordered pairs, duplicates summed, self-loop kept once, sorted rows).
 * Specified in DESIGN.md §6 and reproduced bit-for-bit by oracle/lpa_oracle.c.
 * The graph becomes resident in the context. */
int32_t slpa_gen_rmat(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB,
                      uint32_t tABC, uint64_t seed, int32_t permute, uint64_t perm_key);
int32_t slpa_gen_grid(slpa_ctx *ctx, int64_t rows, int64_t cols, int32_t permute, uint64_t perm_key);
int32_t slpa_gen_kmer(slpa_ctx *ctx, int64_t n, uint32_t keep, uint64_t seed, int32_t permute,
                      uint64_t perm_key);
/* build_graph (graph.py:142-162) from a host edge list; w may be NULL (1.0). */
int32_t slpa_build_graph(slpa_ctx *ctx, int64_t n, int64_t num_edges, const int64_t *src,
                         const int64_t *dst, const double *w, int32_t weights_f64);

/* validate_graph (graph.py:378-403) on the resident graph, checks in the
 * reference's order: code 1 = vertex `*vertex` has a neighbour list that is
 * not strictly increasing, 2 = non-positive weight, 3 = arc set not
 * symmetric (incl. reverse weights), 0 = passed; deg_sum / total are the two
 * sides of the degree-sum identity the caller tests with math.isclose. */
int32_t slpa_validate_graph(slpa_ctx *ctx, int32_t *code, int64_t *vertex, double *deg_sum, double *total);

/* ------------------------------------------------------------ label propagation
 * lpa_run (lpa.py:262-308).  labels_out: host int32[n] or NULL (labels stay
 * resident, fetch with slpa_get_labels).  delta_history: host int64[max_iterations]. */
int32_t slpa_run(slpa_ctx *ctx, const slpa_config *cfg, int32_t *labels_out, int64_t *delta_history,
                 int32_t *iterations, int32_t *converged, slpa_hook_fn hook, void *hook_user);
/* lpa_move (lpa.py:227-259): one sweep on caller state.  labels int32[n] and
 * unprocessed uint8[n] (numpy bool) are read and written back in place. */
int32_t slpa_move(slpa_ctx *ctx, const slpa_config *cfg, int32_t *labels, uint8_t *unprocessed,
                  int32_t pickless, int64_t *changed);
/* Final labels of the last run, by vertex id. */
int32_t slpa_get_labels(slpa_ctx *ctx, int32_t *labels_out);
int32_t slpa_last_run_stats(slpa_ctx *ctx, slpa_run_stats *out);
/* Profiling switch (resets the accumulated profile) and read-out. */
int32_t slpa_set_profiling(slpa_ctx *ctx, int32_t on);
int32_t slpa_get_profile(slpa_ctx *ctx, slpa_profile *out);
/* aux_memory_estimate (lpa.py:311-333) -- the reference's formula. */
int64_t slpa_aux_memory_estimate(int64_t n, int32_t value_bytes, const slpa_config *cfg);

/* ------------------------------------------------------------ metrics
 * _tally / community_stats / modularity (metrics.py:34-74).  labels: host
 * int32[n] by vertex id, or NULL for the resident labels of the last run.
 * sizes/internal/incident may be NULL. */
int32_t slpa_modularity(slpa_ctx *ctx, const int32_t *labels, double *q, int64_t *num_communities,
                        int64_t *sizes, double *internal, double *incident);

/* ------------------------------------------------------------ multi-GPU
 * Contiguous vertex-range partition, one context per rank.
 * The rank holds the rows of [v_begin, v_end) in the global numbering
 * (targets are global ids) plus a full label replica.  A partitioned run is
 * the asynchronous sweep: between sweeps the host all-gathers the owned
 * label ranges and max-reduces the flag arrays (remote entries carry the
 * "neighbour changed" marks of lpa.py:223) -- paper_2411_19901_b200/
 * distributed.py does this with torch.distributed over NCCL. */
int32_t slpa_part_upload(slpa_ctx *ctx, int64_t n, int64_t v_begin, int64_t v_end, const int64_t *row_offsets,
                         const int32_t *targets, const void *weights, int32_t weights_f64);
int32_t slpa_part_gen_rmat(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB,
                           uint32_t tABC, uint64_t seed, int32_t permute, uint64_t perm_key, int64_t v_begin,
                           int64_t v_end);
int32_t slpa_part_info(slpa_ctx *ctx, int64_t *n, int64_t *m_local, int64_t *v_begin, int64_t *v_end);
/* Arc-balanced contiguous ranges of an RMAT graph over `world` ranks:
 * cuts[0..world] (cuts[0] = 0, cuts[world] = n), identical on every rank. */
int32_t slpa_rmat_cuts(slpa_ctx *ctx, int32_t scale, int64_t num_edges, uint32_t tA, uint32_t tAB, uint32_t tABC,
                       uint64_t seed, int32_t permute, uint64_t perm_key, int32_t world, int64_t *cuts);
/* Symmetry of a partitioned graph: every rank reports the 4 hash sums of its
 * rows; the caller sums them over the ranks (mod 2^64) and passes
 * (f1 == r1 && f2 == r2) back.  Deterministic partitioned rounds refuse an
 * unconfirmed or asymmetric graph (SLPA_EUNSUPPORTED). */
int32_t slpa_part_arc_hash(slpa_ctx *ctx, uint64_t *hash4);
int32_t slpa_part_set_symmetric(slpa_ctx *ctx, int32_t symmetric);
/* Device pointers of the label replica (int32[n]) and flag array (uint8[n]). */
int32_t slpa_part_buffers(slpa_ctx *ctx, uint64_t *labels_dptr, uint64_t *flags_dptr);
int32_t slpa_part_begin(slpa_ctx *ctx, const slpa_config *cfg);
int32_t slpa_part_sweep(slpa_ctx *ctx, const slpa_config *cfg, int32_t pickless, int64_t *changed_local);
/* After the exchange: clear the remote (outgoing-mark) flag entries. */
int32_t slpa_part_end_exchange(slpa_ctx *ctx);
/* Deterministic (worker_count == 0) partitioned sweep, one round per call
 * (SURVEY §8(e3)): evaluate the owned flagged (round 0) or dirty vertices and
 * export the dirty marks as bytes; the host then all-gathers the owned ranges
 * of lab_new and MAX-reduces the dirty bytes (views from
 * slpa_part_det_buffers), and slpa_part_det_import folds the global marks
 * back (dirty_total = set marks, identical on every rank; 0 ends the sweep).
 * slpa_part_det_commit closes the sweep (owned changed-vertex count; the
 * flags are then MAX-reduced and slpa_part_end_exchange called as in the
 * asynchronous protocol).  Output is bit-identical to slpa_run. */
int32_t slpa_part_det_buffers(slpa_ctx *ctx, uint64_t *lab_new_dptr, uint64_t *dirty_bytes_dptr);
int32_t slpa_part_det_round(slpa_ctx *ctx, const slpa_config *cfg, int32_t pickless, int32_t round);
int32_t slpa_part_det_import(slpa_ctx *ctx, int64_t *dirty_total);
int32_t slpa_part_det_commit(slpa_ctx *ctx, const slpa_config *cfg, int64_t *changed_local);
/* Rank-local tallies: internal weight (scalar) and device float64[n]
 * incident / int64[n] sizes arrays for an all-reduce; then Q from the
 * reduced incident array and the summed internal weight. */
int32_t slpa_part_tally(slpa_ctx *ctx, double *internal_local, uint64_t *incident_dptr, uint64_t *sizes_dptr);
int32_t slpa_part_modularity(slpa_ctx *ctx, double internal_total, double *q);


/* ------------------------------------------------------------ graph files
 * Parallel host parsers / writers for load_graph / write_edgelist /
 * write_matrix_market (graph.py:165-375).  slpa_edges_parse reads a file into
 * (src, dst, w) entries with the reference's per-line rules and error order
 * (graph.py:165-197 edge lists incl. _remap_ids :200-218; :221-288
 * MatrixMarket, 0-based); the entries then go to slpa_build_graph for the
 * device assembly.  Status codes below; err_line is the 1-based line the
 * reference's message names.  SLPA_IO_EXOTIC: the file needs Python's own
 * text decoding / integer rules (non-ASCII bytes, digit underscores, ids
 * beyond 18 digits) -- the caller parses it itself. */
enum { SLPA_FORMAT_EDGE_LIST = 0, SLPA_FORMAT_MATRIX_MARKET = 1 };
enum {
    SLPA_IO_OK = 0,
    SLPA_IO_EL_FIELDS = 101,      /* "expected 'src dst [weight]', got {aux} fields"  graph.py:173-176 */
    SLPA_IO_EL_NONINT = 102,      /* "non-integer vertex id"                          :177-181 */
    SLPA_IO_EL_NEGATIVE = 103,    /* "negative vertex id"                             :182-183 */
    SLPA_IO_EL_BADWEIGHT = 104,   /* "malformed weight"                               :185-188 */
    SLPA_IO_EL_WEIGHT = 105,      /* "weight must be positive and finite"             :189-190 */
    SLPA_IO_NO_EDGES = 106,       /* "{path}: no edges found"                         :195-196, :285-286 */
    SLPA_IO_MM_HEADER = 110,      /* "not a MatrixMarket matrix file"                 :222-225 */
    SLPA_IO_MM_LAYOUT = 111,      /* :227-228 */
    SLPA_IO_MM_FIELD = 112,       /* :229-230 */
    SLPA_IO_MM_SYMMETRY = 113,    /* :231-232 */
    SLPA_IO_MM_NOSIZE = 114,      /* :242-243 */
    SLPA_IO_MM_SIZE_FIELDS = 115, /* :245-246 */
    SLPA_IO_MM_SIZE_NONINT = 116, /* :247-250 */
    SLPA_IO_MM_NOT_SQUARE = 117,  /* aux x aux2                                       :251-252 */
    SLPA_IO_MM_EMPTY = 118,       /* :253-254 */
    SLPA_IO_MM_ENTRY_FIELDS = 119,/* aux = fields wanted                              :262-263 */
    SLPA_IO_MM_NONINT = 120,      /* :264-268 */
    SLPA_IO_MM_RANGE = 121,       /* :269-270 */
    SLPA_IO_MM_BADVALUE = 122,    /* :272-275 */
    SLPA_IO_MM_VALUE = 123,       /* :276-277 */
    SLPA_IO_MM_COUNT = 124,       /* declared aux, found aux2                         :283-284 */
    SLPA_IO_EXOTIC = 190,
    SLPA_IO_OSERROR = 191,
    SLPA_IO_NOMEM = 192
};
typedef struct slpa_edges slpa_edges;
/* threads <= 0: all hardware threads.  *out is set (free it) whenever the
 * return value is not SLPA_IO_OSERROR. */
int32_t slpa_edges_parse(const char *path, int32_t format, int32_t threads, slpa_edges **out);
int32_t slpa_edges_info(const slpa_edges *e, int64_t *count, int64_t *n, int32_t *remapped, int32_t *err,
                        int64_t *err_line, int64_t *err_aux, int64_t *err_aux2);
/* raw_ids: int64[n] dense id -> id in the file (edge lists with remapped ids). */
int32_t slpa_edges_copy(const slpa_edges *e, int64_t *src, int64_t *dst, double *w, int64_t *raw_ids);
void slpa_edges_free(slpa_edges *e);
/* Canonical writers (graph.py:352-375): text of rows [row_begin, row_end),
 * one "i j w" line per arc with i <= j (lower = 0, edge list) or
 * "i+1 j+1 w" per arc with i >= j (lower = 1, MatrixMarket body), weights as
 * "%.6g".  *buf is malloc'ed (free with slpa_free_buffer). */
int64_t slpa_format_count(int64_t n, const int64_t *offsets, const int32_t *targets, int32_t lower);
int32_t slpa_format_rows(int64_t row_begin, int64_t row_end, const int64_t *offsets, const int32_t *targets,
                         const void *weights, int32_t weights_f64, int32_t lower, int32_t threads, char **buf,
                         int64_t *len);
void slpa_free_buffer(char *buf);

#ifdef __cplusplus
}
#endif
#endif /* SLPA_H */
