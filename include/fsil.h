/*
 * fsil.h -- C ABI of the B200-native linear-time Silhouette (arXiv 2303.14102).
 *
 * Drop-in boundary for the reference fastsil hot path (/root/reference/proj):
 *
 *   reference entry point                                    replaced by
 *   ------------------------------------------------------   ---------------------------------
 *   compute_silhouette(const Dataset&, Metric, Engine, int)   fsil_silhouette (host buffers)
 *     engine.hpp:124-125, engine.cpp:76-92                    fsil_silhouette_device (HBM-resident)
 *   Dataset's fp64 Matrix (dataset.hpp:16-21)                  fsil_silhouette[_device]_f64
 *   validate_and_densify(Matrix, const vector<int>&)          fused into both entries (raw int labels)
 *     dataset.hpp:46, dataset.cpp:26-68
 *   Policy::partial + merge  (aggregate_cluster_stats)        fsil_shard_begin / _dictionary /
 *     engine.hpp:50-80; sqE.cpp:37-63; cos.cpp:39-69           fsil_shard_aggregate + caller all-reduce
 *   Policy::score + finalize_report                           fsil_shard_score + caller all-reduce
 *     engine.hpp:86-115; sqE.cpp:84-108; cos.cpp:90-117;       + fsil_shard_finish
 *     report.cpp:7-47
 *   plan_shards  engine.cpp:8-25                               fsil_plan_shards
 *   assemble_score  report.cpp:7-14                            fsil_assemble_score
 *
 * Features are fp32, N x D row-major (one point per row), byte-compatible
 * with the reference's column-major D x N storage.  Labels are raw int32;
 * dense cluster ids follow first appearance in dataset order (dataset.cpp:41-51).
 * All per-point outputs are in dataset order; every output pointer may be NULL.
 * Exceptions never cross this boundary: every call returns an fsil_status and
 * fsil_last_error() names the violated invariant in the reference's wording.
 * A context is bound to one CUDA device and is not shared by concurrent
 * host threads.  There is no CPU fallback: without a usable sm_100 device
 * fsil_create fails with FSIL_ERR_CUDA.
 */
#ifndef FSIL_H
#define FSIL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSIL_ABI_VERSION 1

typedef enum {
  FSIL_OK = 0,
  FSIL_ERR_IO = 1,               /* fastsil::IoError          (types.hpp:47-50), CLI exit 1 */
  FSIL_ERR_VALIDATION = 2,       /* fastsil::ValidationError  (types.hpp:41-44), CLI exit 2 */
  FSIL_ERR_INVALID_ARGUMENT = 3, /* std::invalid_argument (API misuse)                     */
  FSIL_ERR_CUDA = 4,             /* CUDA runtime / device failure                          */
  FSIL_ERR_NCCL = 5,             /* collective failure (reported by the caller's exchange) */
  FSIL_ERR_INTERNAL = 6,
  FSIL_AGAIN = 7                 /* not an error: fsil_shard_finish after a device dictionary
                                    exchange whose speculated K missed; repeat the protocol */
} fsil_status;

/* Metric (types.hpp:20-24).  FSIL_EUCLID exists only to reproduce the
 * reference's error: the fast engine has no plain-Euclidean path
 * (engine.cpp:89-91). */
typedef enum { FSIL_SQEUCLID = 0, FSIL_COSINE = 1, FSIL_EUCLID = 2 } fsil_metric;

/* Scoring-kernel selection (tests and benchmarks; AUTO picks by cost model). */
/* FSIL_PATH_FP64 evaluates every cluster of every row in fp64 with the reference
 * formulas (the refinement kernel applied to all rows): exact, slow, any shape. */
typedef enum {
  FSIL_PATH_AUTO = 0,
  FSIL_PATH_FFMA = 1,
  FSIL_PATH_TCGEN05 = 2,
  FSIL_PATH_FP64 = 3
} fsil_path;

typedef struct fsil_context fsil_context;

/* Per-call statistics of the last completed call. */
typedef struct {
  int64_t n;               /* rows scored by this context (local rows in shard mode) */
  int32_t d;
  int32_t k;               /* dense clusters */
  int32_t path;            /* fsil_path actually used */
  int32_t agg_path;        /* 1 = warp-private shared-memory, 2 = label-sorted segments, 3 = two-phase batches */
  int64_t flagged_rows;    /* rows re-evaluated by the fp64 argmin refinement kernel */
  int64_t exact_rows;      /* rows whose a_i, b_i, s_i came from the fp64 exact pass (tcgen05 path: all) */
  int64_t kernel_launches; /* kernels launched by the last call */
  float ms_densify, ms_aggregate, ms_score, ms_refine, ms_finalize; /* device time, 0 unless timing on */
  float ms_score_kernel;   /* the scoring kernel alone (ms_score minus its operand preparation) */
  int64_t pair_rows;       /* rows whose neighbour was one of two certified candidates, decided in fp64 */
  int32_t tc_mmas;         /* tensor-core MMAs per 16-deep K step of the pass that scored every row:
                              3 (fp16x3), 2 (the two-level certificate's first level); 0 otherwise */
  int32_t tc_threshold;    /* 1: the tensor-core pass ran in threshold mode (comparison inside the MMA) */
  int64_t rescored_rows;   /* two-level certificate: rows re-scored at three-MMA precision */
} fsil_stats;

fsil_status fsil_create(fsil_context** ctx, int device);
void fsil_destroy(fsil_context* ctx);
const char* fsil_last_error(const fsil_context* ctx);
int fsil_abi_version(void);

/* Stream used by every kernel of this context (cudaStream_t).  NULL selects a
 * context-owned non-blocking stream (the default); to order with work on the
 * legacy default stream -- e.g. a framework's stream 0 and collectives issued
 * on it -- pass cudaStreamLegacy ((void*)0x1), not NULL. */
fsil_status fsil_set_stream(fsil_context* ctx, void* stream);
fsil_status fsil_set_path(fsil_context* ctx, int path);
/* Per-phase CUDA-event timing on the context stream (adds no syncs beyond the call's own). */
fsil_status fsil_set_timing(fsil_context* ctx, int enabled);
fsil_status fsil_get_stats(const fsil_context* ctx, fsil_stats* out);

/*
 * Whole-dataset Silhouette on host buffers: compute_silhouette(
 * validate_and_densify(X, labels), metric, Engine::Fast).  Copies X and
 * labels to HBM, runs the device pipeline, copies results back.
 *   X [n*d] fp32 row-major, labels [n] raw int32.
 *   s, a, b [n] fp64; neighbour, own [n] dense ids; mean = S;
 *   k_out = K; dense_to_raw [K] (capacity n) = raw label of each dense id.
 */
fsil_status fsil_silhouette(fsil_context* ctx, int metric, const float* X, const int32_t* labels,
                            int64_t n, int32_t d, double* s, int32_t* neighbour, int32_t* own,
                            double* a, double* b, double* mean, int32_t* k_out,
                            int32_t* dense_to_raw);

/* Same with device-resident inputs and device-resident per-point outputs
 * (mean, k_out and dense_to_raw are host pointers).  This is the entry the
 * benchmark times: data already in HBM, as in the reference's timed window
 * (engine.hpp:107-113). */
fsil_status fsil_silhouette_device(fsil_context* ctx, int metric, const float* dX,
                                   const int32_t* dlabels, int64_t n, int32_t d, double* ds,
                                   int32_t* dneighbour, int32_t* down, double* da, double* db,
                                   double* mean, int32_t* k_out, int32_t* dense_to_raw);

/*
 * fp64 front end: the same calls on fp64 features -- the reference's
 * own Matrix (Eigen::MatrixXd, D x N column-major == N x D row-major, dataset.hpp:16-21).
 * Aggregation, the fp64 refinement and the exact a/b recompute read the fp64 values;
 * the fast scoring pass reads their fp32 rounding, with that rounding (u relative)
 * added to its certified error bounds.  Scoring runs on the tensor cores (or in fp64
 * where the shape has no tensor-core tiling); FSIL_PATH_FFMA is unavailable here.
 */
fsil_status fsil_silhouette_f64(fsil_context* ctx, int metric, const double* X, const int32_t* labels,
                                int64_t n, int32_t d, double* s, int32_t* neighbour, int32_t* own,
                                double* a, double* b, double* mean, int32_t* k_out, int32_t* dense_to_raw);
fsil_status fsil_silhouette_device_f64(fsil_context* ctx, int metric, const double* dX,
                                       const int32_t* dlabels, int64_t n, int32_t d, double* ds,
                                       int32_t* dneighbour, int32_t* down, double* da, double* db,
                                       double* mean, int32_t* k_out, int32_t* dense_to_raw);

/*
 * The Theta(N^2 D) engine (naive_silhouette, naive.cpp:30-71) on the GPU:
 * every pairwise distance in fp64, for cross-checks (the reference's `compare`) and for
 * FSIL_EUCLID, which has no linear-time decomposition.  Same validation, outputs and
 * errors as fsil_silhouette_f64; meant for small N (K x 128 + 64 x D doubles of shared
 * memory per block).
 */
fsil_status fsil_silhouette_naive(fsil_context* ctx, int metric, const double* X, const int32_t* labels,
                                  int64_t n, int32_t d, double* s, int32_t* neighbour, int32_t* own,
                                  double* a, double* b, double* mean, int32_t* k_out, int32_t* dense_to_raw);

/*
 * Sharded (multi-GPU, one process per GPU) protocol.  Rank r owns the
 * contiguous global rows [row_offset, row_offset + n_local) (plan_shards
 * semantics).  The caller performs the three exchanges between phases with
 * its own collective library (NCCL via torch.distributed in this repo):
 *
 *   1. fsil_shard_begin            -> local dictionary of distinct raw labels
 *      fsil_shard_get_dictionary   -> (raw label, first global row) pairs
 *      [exchange: all-gather; merge by min first row; order by first row]
 *      fsil_shard_set_dictionary   <- global raw labels in dense order
 *   2. fsil_shard_aggregate        -> device fp64 buffer of K*(D+2) (sqeuclid)
 *                                     or K*(D+1) (cosine) sums, and a device
 *                                     int64[2] validation word
 *      [exchange: all-reduce SUM of the stats buffer, MIN of the int64 word]
 *   3. fsil_shard_score            -> device fp64 [2] = {sum of s_i, flagged rows}
 *      [exchange: all-reduce SUM]
 *      fsil_shard_finish           -> validates the reduced words, mean = sum / N
 */
fsil_status fsil_shard_begin(fsil_context* ctx, int metric, const float* dX,
                             const int32_t* dlabels, int64_t n_local, int32_t d,
                             int64_t row_offset, int64_t n_global, int64_t* n_distinct);
/* fsil_shard_begin on fp64 features (the fp64 front end above). */
fsil_status fsil_shard_begin_f64(fsil_context* ctx, int metric, const double* dX,
                                 const int32_t* dlabels, int64_t n_local, int32_t d,
                                 int64_t row_offset, int64_t n_global, int64_t* n_distinct);
fsil_status fsil_shard_get_dictionary(fsil_context* ctx, int32_t* raw_labels, int64_t* first_rows);
fsil_status fsil_shard_set_dictionary(fsil_context* ctx, const int32_t* raw_in_dense_order,
                                      int32_t k);
fsil_status fsil_shard_aggregate(fsil_context* ctx, double** d_stats, int64_t* stats_len,
                                 int64_t** d_checks);
fsil_status fsil_shard_score(fsil_context* ctx, double* ds, int32_t* dneighbour, int32_t* down,
                             double* da, double* db, double** d_partial);
fsil_status fsil_shard_finish(fsil_context* ctx, double* mean);

/*
 * The same protocol with the dictionary exchange on the device (no host round trip):
 *   fsil_shard_begin_device        -> device buffer of `capacity` (label, first global row)
 *                                     int64 pairs (unused: row -1), identical capacity on
 *                                     every rank; xtype 0 = fp32 features, 1 = fp64
 *   [exchange: all-gather the buffers of all ranks, rank order]
 *   fsil_shard_set_dictionary_device <- the gathered nranks x capacity pairs: merged on the
 *                                     device (first appearance)
 * then fsil_shard_aggregate / _score / _finish as above.
 *
 * K speculation.  The kernels after the dictionary are sized by K.  Rather than wait for
 * the merged count, set_dictionary_device launches them for the previous call's global K
 * (identical on every rank), so the protocol's only host sync is in fsil_shard_finish.
 * finish checks the count; if it differs, every rank returns FSIL_AGAIN and the caller
 * repeats the protocol from fsil_shard_begin_device (the repeat waits for the count).  The
 * single-GPU entries speculate the same way and repeat internally.  FSIL_SPECULATE=0 in the
 * environment at fsil_create turns it off.
 */
fsil_status fsil_shard_begin_device(fsil_context* ctx, int metric, const void* dX, int xtype,
                                    const int32_t* dlabels, int64_t n_local, int32_t d,
                                    int64_t row_offset, int64_t n_global, int64_t** d_entries,
                                    int64_t* capacity);
fsil_status fsil_shard_set_dictionary_device(fsil_context* ctx, const int64_t* d_gathered,
                                             int32_t nranks, int64_t capacity);

/* plan_shards (engine.cpp:8-25): writes w' = min(w, n) (begin, end) pairs. */
fsil_status fsil_plan_shards(int64_t n, int32_t requested, int64_t* ranges, int32_t* num_shards);
/* assemble_score (report.cpp:7-14). */
fsil_status fsil_assemble_score(double a, double b, double* s);

#ifdef __cplusplus
}
#endif

#endif /* FSIL_H */
