/*
 * fsil_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference fastsil hot path (arXiv 2303.14102), used as
 * the parity checker for the B200 product path and as the CPU baseline in
 * bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product (libfsil.so) never
 * links or calls it.
 *
 * Parity status: pinned bit for bit to the reference itself.  oracle/Makefile
 * `ref` compiles the reference's own .cpp files (unmodified, from
 * /root/reference/proj/src) against a committed Eigen-API shim into
 * oracle/_ref/libfsil_ref.so; tests/test_oracle.py checks that this
 * restatement returns identical a, b, s, own, neighbour and mean bits on every
 * shape it runs (the reductions restate Eigen 3.4.0's SSE2 redux order).  It is
 * also checked against SPEC.md's goldens, the naive O(N^2 D) engine and
 * scikit-learn's silhouette_samples (tests/golden/).
 */
#ifndef FSIL_ORACLE_H
#define FSIL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror include/fsil.h (and the reference's exception classes). */
enum {
  ORC_OK = 0,
  ORC_ERR_IO = 1,
  ORC_ERR_VALIDATION = 2,       /* fastsil::ValidationError (types.hpp:41-44) */
  ORC_ERR_INVALID_ARGUMENT = 3, /* std::invalid_argument                    */
  ORC_ERR_INTERNAL = 6
};

/* Metric / Engine enums: types.hpp:20-29. */
enum { ORC_SQEUCLID = 0, ORC_COSINE = 1, ORC_EUCLID = 2 };
enum { ORC_FAST = 0, ORC_NAIVE = 1 };

/*
 * compute_silhouette(validate_and_densify(X, labels), metric, engine, shards)
 * (engine.cpp:76-92, dataset.cpp:63-68).  X is N x D row-major fp64, which is
 * byte-identical to the reference's column-major D x N Eigen::MatrixXd.
 * Outputs (each nullable): a, b, s [N]; own, neighbour [N] dense ids;
 * mean; k_out; dense_to_raw [K] (capacity N); wall_ms = the reference's
 * run_two_phase window (engine.hpp:107-113).
 */
int orc_silhouette(int metric, int engine, const double* X, const int32_t* labels, int64_t n,
                   int64_t d, int shards, double* a, double* b, double* s, int32_t* own,
                   int32_t* neighbour, double* mean, int32_t* k_out, int32_t* dense_to_raw,
                   double* wall_ms, char* err, size_t errlen);

/* Same, fp32 input widened exactly to fp64 before the timed window. */
int orc_silhouette_f32(int metric, int engine, const float* X, const int32_t* labels, int64_t n,
                       int64_t d, int shards, double* a, double* b, double* s, int32_t* own,
                       int32_t* neighbour, double* mean, int32_t* k_out, int32_t* dense_to_raw,
                       double* wall_ms, char* err, size_t errlen);

/*
 * Phase 1 only: merged per-cluster statistics (aggregate_cluster_stats,
 * engine.hpp:50-80) over a densified dataset.  counts[K] int64;
 * sums[K*D] (Y_k for sqeuclid, Omega_k for cosine, cluster-major);
 * psi[K] (sqeuclid only; may be NULL for cosine).
 */
int orc_aggregate_f32(int metric, const float* X, const int32_t* labels, int64_t n, int64_t d,
                      int shards, int64_t* counts, double* sums, double* psi, int32_t* k_out,
                      char* err, size_t errlen);

/*
 * Phase 2 on a row subset against given merged stats (score_range,
 * squared_euclidean.cpp:84-108 / cosine.cpp:90-117).  rows[m] are indices into
 * X; dense[] are dense labels for all N rows.  Used to verify sampled rows of
 * configs too large for a full CPU run: s_i depends only on (x_i, label_i,
 * global stats).
 */
int orc_score_rows_f32(int metric, const float* X, const int32_t* dense, int64_t n, int64_t d,
                       int32_t k, const int64_t* counts, const double* sums, const double* psi,
                       const int64_t* rows, int64_t m, double* a, double* b, double* s,
                       int32_t* neighbour, char* err, size_t errlen);

/* Same on `threads` std::threads (0 = all); rows == NULL scores rows [0, m). */
int orc_score_rows_mt_f32(int metric, const float* X, const int32_t* dense, int64_t n, int64_t d,
                          int32_t k, const int64_t* counts, const double* sums, const double* psi,
                          const int64_t* rows, int64_t m, int threads, double* a, double* b,
                          double* s, int32_t* neighbour, char* err, size_t errlen);

/* aggregate_cluster_stats over labels that are already dense ids in [0, k)
 * (skips the string densify, which is impractical at 1e8 rows); same block
 * plan and fold as orc_aggregate_f32.  Used to pin full-size configs. */
int orc_aggregate_dense_f32(int metric, const float* X, const int32_t* dense, int64_t n, int64_t d,
                            int32_t k, int shards, int64_t* counts, double* sums, double* psi,
                            char* err, size_t errlen);

/* plan_shards (engine.cpp:8-25): writes w' (begin,end) pairs, returns w'. */
int orc_plan_shards(int64_t n, int requested, int64_t* ranges, int* num_shards, char* err,
                    size_t errlen);

/* assemble_score (report.cpp:7-14). */
int orc_assemble_score(double a, double b, double* s, char* err, size_t errlen);

/* default_shards (engine.cpp:27-30). */
int orc_default_shards(void);

#ifdef __cplusplus
}
#endif

#endif /* FSIL_ORACLE_H */
