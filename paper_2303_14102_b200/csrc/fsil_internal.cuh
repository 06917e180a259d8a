// fsil_internal.cuh -- shared device/host definitions for libfsil (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "fsil.h"

namespace fsil {

// ---- errors crossing the internal C++ layers (converted to fsil_status at the C ABI) ----
struct Error : std::runtime_error {
  fsil_status status;
  Error(fsil_status st, const std::string& msg) : std::runtime_error(msg), status(st) {}
};
[[noreturn]] inline void fail(fsil_status st, const std::string& msg) { throw Error(st, msg); }

#define FSIL_CUDA(call)                                                                    \
  do {                                                                                     \
    cudaError_t e__ = (call);                                                              \
    if (e__ != cudaSuccess)                                                                \
      ::fsil::fail(FSIL_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__));    \
  } while (0)

#define FSIL_LAUNCHED(ctx)                                                                 \
  do {                                                                                     \
    cudaError_t e__ = cudaGetLastError();                                                  \
    if (e__ != cudaSuccess)                                                                \
      ::fsil::fail(FSIL_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e__)); \
    ++(ctx)->launches;                                                                     \
    if ((ctx)->debug_sync) {  /* FSIL_DEBUG_SYNC=1: name the kernel that faults */           \
      e__ = cudaStreamSynchronize((ctx)->stream);                                            \
      if (e__ != cudaSuccess)                                                                \
        ::fsil::fail(FSIL_ERR_CUDA, std::string("kernel at " __FILE__ ":") +                 \
                                        std::to_string(__LINE__) + ": " + cudaGetErrorString(e__)); \
    }                                                                                        \
  } while (0)

constexpr int kNumSMs = 148;
// int index in the context's 64-byte counters block (zeroed by every dictionary pass) of
// the K-speculation miss flag the densify kernels raise for the scoring kernels
constexpr int kAbortWord = 10;  // B200; the context re-reads the real count

// ---- grow-only device scratch -----------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  void ensure(size_t want) {
    if (want <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t cap = want < 4096 ? 4096 : want + want / 8;
    FSIL_CUDA(cudaMalloc(&p, cap));
    bytes = cap;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// Layout of the fp64 cluster-statistics buffer (the all-reduce payload):
//   sqeuclid: [count K][psi K][sums K*D]    -> K*(D+2)
//   cosine  : [count K][sums K*D]           -> K*(D+1)
struct StatsLayout {
  int metric;
  int64_t k, d;
  int64_t count_off() const { return 0; }
  int64_t psi_off() const { return k; }
  int64_t sums_off() const { return metric == FSIL_SQEUCLID ? 2 * k : k; }
  int64_t len() const { return sums_off() + k * d; }
};

// Derived per-cluster constants consumed by the scoring kernels.
struct Derived {
  float* mu32;       // [K][dp] fp32: Y_k/n_k (sqeuclid) or Omega_k/n_k (cosine), zero padded
  float* p32;        // [K] sqeuclid: psi_k/n_k in fp32
  double* nk;        // [K] counts as fp64
  float* bound;      // [4]: max ||mu_k||, max p_k, 0, 0 (fp32, rounded up)
};

// Validation word, all-reduced with MIN across ranks.
//   [0] first non-finite element as global row*D + dim (INT64_MAX if none)
//   [1] first zero-norm row (cosine only; INT64_MAX if none)
constexpr int64_t kNone = INT64_MAX;

// Per-call words the host reads back, written by kernels straight into mapped pinned
// memory (one stream sync, no pageable copies).
struct HostSummary {
  int64_t overflow;   // densify: hash table overflowed (retry with a larger table)
  int64_t count;      // densify: distinct labels (K)
  int64_t checks[2];  // validation word (after the caller's MIN all-reduce in shard mode)
  int64_t missing;    // a row's label absent from the dictionary
  int64_t pad;
  double result[4];   // sum of s_i, flagged rows, exact rows, certified-pair rows
};

}  // namespace fsil

// ---- context (C ABI handle) ----------------------------------------------------------------
struct fsil_context {
  int device = 0;
  int num_sms = fsil::kNumSMs;
  size_t smem_optin = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int path = FSIL_PATH_AUTO;
  bool timing = false;
  std::string last_error;
  int64_t launches = 0;
  fsil_stats stats{};

  // shard/call state
  int metric = FSIL_SQEUCLID;
  const float* X = nullptr;       // fp32 features the scoring kernels read
  const double* X64 = nullptr;    // fp64 front end: the caller's features (aggregation, exact parts)
  const int32_t* labels = nullptr;
  int64_t n = 0, n_global = 0, row_offset = 0;
  int32_t d = 0, k = 0;
  int64_t dp = 0;  // d rounded up to a multiple of 4
  int64_t n_distinct = 0;
  int agg_path = 0;
  int score_path = 0;
  int phase = 0;  // 0 idle, 1 begun, 2 dictionary set, 3 aggregated, 4 scored

  // scratch (grow-only)
  fsil::DevBuf ht_keys, ht_vals, ht_dense, dict_labels, dict_rows, dict_sorted, counters;
  const int32_t* dict_sorted_labels = nullptr;  // device: raw labels in dense order (single GPU)
  fsil::DevBuf dense;          // [n] int32 dense labels
  fsil::DevBuf stats_buf;      // fp64 stats (all-reduce payload)
  fsil::DevBuf checks;         // int64[2] validation word
  fsil::DevBuf partials;       // aggregation block partials
  fsil::DevBuf sort_tmp, sort_keys, sort_vals, iota;  // label-sorted aggregation
  fsil::DevBuf seg_start, piece_start;
  fsil::DevBuf mu32, p32, nk, bound;
  fsil::DevBuf s_tmp;          // s when the caller passes no s pointer
  fsil::DevBuf tile_sum, tile_flag, flag_rows, flag_count;
  fsil::DevBuf refine_part, refine_cnt;  // split tiled refinement: slice minima, row-tile tickets
  fsil::DevBuf result;         // double[4]: sum_s, flagged, ... (shard partial)
  fsil::DevBuf group_sum;
  fsil::DevBuf xmax;           // float: max |x| of this shard (tensor-core operand scaling)
  fsil::DevBuf tc_b;           // fp16 cluster-mean pieces + column bias (tcgen05 path)
  fsil::DevBuf nb_tmp;                   // neighbours when the caller passes no neighbour pointer
  fsil::DevBuf sub_x, sub_i;             // two-level certificate: the level-1 uncertain rows (x, ids)
  fsil::DevBuf cand_rows;                // threshold mode: rows with 3-4 candidate neighbours (int4 records)
  fsil::DevBuf thr_nn, thr_t;            // threshold mode: candidate clusters per cluster, t slots per row
  int32_t tc_thr = 0;                    // this call's tensor-core pass ran in threshold mode (stats)
  int32_t tc_mmas = 0;                   // MMAs per K step of this call's tensor-core pass (stats)
  int64_t rescored = 0;                  // two-level certificate: rows re-scored at three MMAs
  fsil::DevBuf pair_rows, pair_count;    // tcgen05 top-3: rows resolved as a certified pair
  fsil::DevBuf a_scratch;                // tcgen05 streaming mode: per-CTA converted A chunks
  fsil::DevBuf x32;                      // fp64 front end: rounded fp32 copy for the fast pass
  fsil::DevBuf xi_rows;                  // fp64 ||x||^2 per row, written by the batched aggregation
  bool xi_valid = false;                 // xi_rows holds this call's rows (scoring reads them)
  fsil::DevBuf xbuf;                     // sharded protocol: device dictionary exchange entries
  fsil::DevBuf xt_keys, xt_vals, xt_dense;  // ... and the global-dictionary table (own epochs)
  int64_t xt_cap = 0;
  // K speculation (densify_local / densify_exchange_set): kernels launched for the previous
  // call's K, checked by finish() against this call's count.
  bool speculate = true;   // FSIL_SPECULATE=0 disables
  bool debug_sync = false;  // FSIL_DEBUG_SYNC=1: synchronise and check after every launch
  bool fuse_post = true;    // FSIL_FUSE_POST=0: separate exact / refine / tile-group launches
  bool k_spec = false;     // this call speculated
  bool spec_big = false;   // ... with the multi-block ordering launched
  bool spec_missed = false;
  bool spec_block_once = false;  // the retry after a miss waits for the count
  int32_t* d2r_host = nullptr;    // pinned staging of dense_to_raw (copied out once K is confirmed)
  int64_t d2r_cap = 0;
  int64_t spec_cap_x = 0;
  uint32_t xt_epoch = 0;
  // host staging for fsil_silhouette (pageable -> pinned)
  fsil::DevBuf hX, hL;         // device copies of host inputs
  fsil::DevBuf o_s, o_nb, o_own, o_a, o_b;
  int64_t ht_cap = 0;        // hash-table slots wanted for the next call
  int64_t ht_alloc_cap = 0;  // slots of the current (zero-initialised) table
  uint32_t ht_epoch = 0;     // epoch of the last densify (table entries are epoch-tagged)
  int64_t k_last = 0;        // K of the previous call (picks the ordering path)
  int64_t k_global_last = 0; // sharded: the previous call's global K (sizes the device exchange)
  bool local_call = false;   // single-GPU call (fsil_silhouette[_device]), not the shard protocol
  bool summary_packed = false;  // this call's HostSummary already written on the device
  bool naive_call = false;      // fsil_silhouette_naive: the Theta(N^2 D) engine
  fsil::HostSummary* hsum = nullptr;  // mapped pinned (host view)
  fsil::HostSummary* dsum = nullptr;  // device view of the same memory
  cudaEvent_t ev[8] = {};
  bool ev7_recorded = false;  // ev[7] marks the scoring kernel's own launch (timing runs)
  bool pdl = true;             // programmatic dependent launch on the hot chain (FSIL_PDL=0: off)
};

namespace fsil {

// Launch on the context stream with programmatic dependent launch: the kernel may be
// scheduled while its stream predecessor drains (hiding the launch gap between the
// chain's kernels).  Every kernel launched this way calls griddep_wait() before touching
// memory, so it still observes everything its predecessors wrote.
template <typename... KArgs, typename... Args>
inline void launch_pdl(fsil_context* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FSIL_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
  FSIL_LAUNCHED(c);
}

// kernels.cu entry points (host launchers), all async on ctx->stream
void densify_collect(fsil_context* c);     // fills ctx->n_distinct (syncs)
void densify_local(fsil_context* c);       // single GPU: dense ids + K, one sync
void densify_assign_and_map(fsil_context* c, const int32_t* raw_in_dense_order, int32_t k);
int64_t* densify_exchange_begin(fsil_context* c, int64_t cap_x);
void densify_exchange_set(fsil_context* c, const int64_t* gathered, int nranks, int64_t cap_x);
void exchange_grow(fsil_context* c, int64_t cap_x);
void aggregate(fsil_context* c);           // stats_buf + checks
void derive(fsil_context* c);              // mu32, p32, nk, bound
void score(fsil_context* c, double* s, int32_t* nb, int32_t* own, double* a, double* b);
void finalize_partial(fsil_context* c, double* s);  // result[0] = sum s, result[1] = flagged
void score_tc(fsil_context* c, double* s, int32_t* nb, int32_t* own, double* a, double* b);
bool tc_supported(const fsil_context* c);

}  // namespace fsil
