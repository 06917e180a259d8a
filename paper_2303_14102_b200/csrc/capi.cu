// capi.cu -- the C ABI (include/fsil.h): context, validation in the reference's
// order and wording, the single-GPU pipeline and the sharded protocol.
//
// Pipeline per call (all on ctx->stream; two host syncs: K after densify, and
// the final scalar words):
//   K0 densify (densify.cu) -> K1 aggregate (aggregate.cu) -> derive ->
//   K2 score_ffma | K3 score_tc -> K4 refine -> K5 tile-group sum (finalize.cu)
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include "fsil_internal.cuh"
#include "score_common.cuh"

namespace fsil {

void score_ffma(fsil_context* c, const ScoreParams& p);
int64_t ffma_tiles(int64_t n);
void score_naive(fsil_context* c, const ScoreParams& p);
int64_t naive_tiles(int64_t n, int* tile_rows);
bool ffma_supported(const fsil_context* c);
void flag_all(fsil_context* c, const ScoreParams& p, int tile_rows);
void exact_pass(fsil_context* c, const ScoreParams& p, bool local);
void refine(fsil_context* c, const ScoreParams& p);
void finalize_sum(fsil_context* c, const ScoreParams& p, int64_t ntiles, int tile_rows, bool local);
bool post_fused(fsil_context* c, const ScoreParams& p, int64_t ntiles, int tile_rows, bool local);
bool tc_supported(const fsil_context* c);
int64_t tc_tiles(const fsil_context* c, int* tile_rows);
void score_tc(fsil_context* c, const ScoreParams& p);

namespace {

void record(fsil_context* c, int i) {
  if (i == 3) c->ev7_recorded = false;  // the scoring phase starts: its kernel mark is re-taken
  if (c->timing) FSIL_CUDA(cudaEventRecord(c->ev[i], c->stream));
}

void check_metric(int metric) {
  if (metric != FSIL_SQEUCLID && metric != FSIL_COSINE && metric != FSIL_EUCLID)
    fail(FSIL_ERR_INVALID_ARGUMENT, "unknown metric code " + std::to_string(metric));
}

// validate_and_densify's shape checks (dataset.cpp:29-34).
void check_shape(int64_t n_global, int64_t d) {
  if (n_global < 2)
    fail(FSIL_ERR_VALIDATION, "dataset needs at least 2 points, got " + std::to_string(n_global));
  if (d < 1) fail(FSIL_ERR_VALIDATION, "dataset needs at least 1 feature dimension");
}

// fp64 front end: the fast scoring pass reads a rounded fp32 copy
__global__ void to_f32_kernel(const double* __restrict__ in, float* __restrict__ out, int64_t count) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<float>(in[i]);
}

// dX: fp32 (x64 = false) or fp64 (x64 = true) features, n_local x d row-major.
void setup(fsil_context* c, int metric, const void* dX, bool x64, const int32_t* dlabels, int64_t n_local,
           int32_t d, int64_t row_offset, int64_t n_global) {
  check_metric(metric);
  check_shape(n_global, d);
  if (n_local < 0 || row_offset < 0 || row_offset + n_local > n_global)
    fail(FSIL_ERR_INVALID_ARGUMENT, "shard rows outside the dataset");
  if (n_local > 0 && (!dX || !dlabels)) fail(FSIL_ERR_INVALID_ARGUMENT, "null input pointer");
  FSIL_CUDA(cudaSetDevice(c->device));
  c->metric = metric;
  if (x64) {
    c->X64 = static_cast<const double*>(dX);
    const int64_t count = n_local * static_cast<int64_t>(d);
    c->x32.ensure(std::max<int64_t>(count, 1) * sizeof(float));
    if (count > 0) {
      to_f32_kernel<<<static_cast<unsigned>(std::min<int64_t>((count + 255) / 256, int64_t(c->num_sms) * 16)), 256, 0,
                      c->stream>>>(c->X64, c->x32.as<float>(), count);
      FSIL_LAUNCHED(c);
    }
    c->X = c->x32.as<float>();
  } else {
    c->X64 = nullptr;
    c->X = static_cast<const float*>(dX);
  }
  c->labels = dlabels;
  c->n = n_local;
  c->n_global = n_global;
  c->row_offset = row_offset;
  c->d = d;
  c->dp = (static_cast<int64_t>(d) + 3) / 4 * 4;
  c->k = 0;
  c->k_spec = false;
  c->spec_missed = false;
  c->stats = fsil_stats{};
  c->tc_mmas = 0;
  c->tc_thr = 0;
  c->rescored = 0;
  record(c, 0);
}

void begin(fsil_context* c, int metric, const void* dX, bool x64, const int32_t* dlabels, int64_t n_local,
           int32_t d, int64_t row_offset, int64_t n_global) {
  c->launches = 0;
  setup(c, metric, dX, x64, dlabels, n_local, d, row_offset, n_global);
  c->local_call = false;
  densify_collect(c);
  c->phase = 1;
}

void set_dictionary(fsil_context* c, const int32_t* raw, int32_t k) {
  if (c->phase < 1) fail(FSIL_ERR_INVALID_ARGUMENT, "fsil_shard_begin must come first");
  if (k < 1 || (k > 0 && !raw)) fail(FSIL_ERR_INVALID_ARGUMENT, "empty dictionary");
  c->k = k;
  densify_assign_and_map(c, raw, k);
  record(c, 1);
  c->phase = 2;
}

void do_aggregate(fsil_context* c) {
  if (c->phase < 2) fail(FSIL_ERR_INVALID_ARGUMENT, "dictionary not set");
  // Plain euclidean has no aggregable decomposition; the dataset is still
  // validated first, as the reference builds the Dataset before dispatching.
  const int saved = c->metric;
  if (c->metric == FSIL_EUCLID) c->metric = FSIL_SQEUCLID;
  aggregate(c);
  c->metric = saved;
  record(c, 2);
  c->phase = 3;
}

ScoreParams make_params(fsil_context* c, double* s, int32_t* nb, int32_t* own, double* a,
                        double* b) {
  ScoreParams p{};
  p.X = c->X;
  p.X64 = c->X64;
  p.dense = c->dense.as<int32_t>();
  p.n = c->n;
  p.d = c->d;
  p.dp = static_cast<int>(c->dp);
  p.k = c->k;
  p.mu32 = c->mu32.as<float>();
  p.p32 = c->p32.as<float>();
  p.stats = c->stats_buf.as<double>();
  p.nk = c->nk.as<double>();
  p.bound = c->bound.as<float>();
  p.abort = c->counters.as<int>() + kAbortWord;
  if (!s) {
    c->s_tmp.ensure(std::max<int64_t>(c->n, 1) * sizeof(double));
    s = c->s_tmp.as<double>();
  }
  p.s = s;
  if (!nb) {  // the scoring pass nominates into it, the exact pass reads it back
    c->nb_tmp.ensure(std::max<int64_t>(c->n, 1) * sizeof(int32_t));
    nb = c->nb_tmp.as<int32_t>();
  }
  p.nb = nb;
  p.own = own;
  p.a = a;
  p.b = b;
  return p;
}

void do_score(fsil_context* c, double* s, int32_t* nb, int32_t* own, double* a, double* b) {
  if (c->phase < 3) fail(FSIL_ERR_INVALID_ARGUMENT, "aggregate must come before score");
  c->result.ensure(4 * sizeof(double));  // zeroed with the counters by agg_init
  c->phase = 4;
  if (c->k < 2 || (c->metric == FSIL_EUCLID && !c->naive_call) || c->n == 0) {  // reported by finish
    record(c, 3); record(c, 4); record(c, 5);
    return;
  }
  if (c->naive_call) {  // the Theta(N^2 D) engine: every pair in fp64, nothing to refine
    ScoreParams p = make_params(c, s, nb, own, a, b);
    int tile_rows = 128;
    const int64_t ntiles = naive_tiles(c->n, &tile_rows);
    c->tile_sum.ensure(std::max<int64_t>(ntiles, 1) * sizeof(double));
    c->tile_flag.ensure(std::max<int64_t>(ntiles, 1) * sizeof(int32_t));
    c->flag_count.ensure(sizeof(unsigned long long));
    FSIL_CUDA(cudaMemsetAsync(c->flag_count.p, 0, sizeof(unsigned long long), c->stream));
    p.tile_sum = c->tile_sum.as<double>();
    p.tile_flag = c->tile_flag.as<int32_t>();
    p.flag_count = c->flag_count.as<unsigned long long>();
    record(c, 3);
    score_naive(c, p);
    c->score_path = 0;
    record(c, 4);
    record(c, 5);
    finalize_sum(c, p, ntiles, tile_rows, c->local_call);
    c->summary_packed = c->local_call;
    return;
  }
  derive(c);
  ScoreParams p = make_params(c, s, nb, own, a, b);
  int use = c->path;
  // the FFMA kernel's own fp64 a/b recompute reads the fp32 features: not exact on
  // the fp64 front end, which therefore scores on the tensor cores or in fp64
  const bool tc_ok = tc_supported(c), ffma_ok = !c->X64 && ffma_supported(c);
  if (use == FSIL_PATH_AUTO) {
    // Measured crossover (profiles/): the tcgen05 kernel wins once the contraction
    // has ~2e7 row-cluster pairs (C2: 116 us vs 207 us FFMA); below that its fixed
    // costs (operand prep, one scale readback) dominate and FFMA wins (C1).
    const double pairs = static_cast<double>(c->n) * c->k;
    if (tc_ok && (pairs >= 1.5e7 || !ffma_ok || c->k > 32)) use = FSIL_PATH_TCGEN05;
    else if (ffma_ok) use = FSIL_PATH_FFMA;
    else use = FSIL_PATH_FP64;
  }
  if (use == FSIL_PATH_TCGEN05 && !tc_ok)
    fail(FSIL_ERR_INVALID_ARGUMENT, "tcgen05 scoring path unavailable for this shape (d=" +
                                        std::to_string(c->d) + ", k=" + std::to_string(c->k) +
                                        ", smem optin " + std::to_string(c->smem_optin) + ")");
  if (use == FSIL_PATH_FFMA && !ffma_ok)
    fail(FSIL_ERR_INVALID_ARGUMENT, c->X64 ? "FFMA scoring path unavailable for fp64 features"
                                           : "FFMA scoring path unavailable for this shape (D too large)");
  int tile_rows = 256;
  const int64_t ntiles = use == FSIL_PATH_TCGEN05 ? tc_tiles(c, &tile_rows) : ffma_tiles(c->n);
  c->tile_sum.ensure(std::max<int64_t>(ntiles, 1) * sizeof(double));
  c->tile_flag.ensure(std::max<int64_t>(ntiles, 1) * sizeof(int32_t));
  c->flag_rows.ensure(std::max<int64_t>(c->n, 1) * sizeof(int32_t));
  c->flag_count.ensure(sizeof(unsigned long long));  // zeroed by agg_init
  p.tile_sum = c->tile_sum.as<double>();
  p.tile_flag = c->tile_flag.as<int32_t>();
  p.flag_rows = c->flag_rows.as<int32_t>();
  p.flag_count = c->flag_count.as<unsigned long long>();
  record(c, 3);
  if (use == FSIL_PATH_TCGEN05) score_tc(c, p);
  else if (use == FSIL_PATH_FFMA) score_ffma(c, p);
  else flag_all(c, p, tile_rows);
  c->score_path = use;
  record(c, 4);
  // single GPU: the final kernel also fills the mapped host summary (no pack launch)
  if (use == FSIL_PATH_TCGEN05) {
    // the tensor-core pass only nominates neighbours: refinement of the uncertain rows,
    // then every row's a_i, b_i, s_i in fp64 and the deterministic total
    exact_pass(c, p, c->local_call);
    record(c, 5);
  } else if (c->fuse_post && post_fused(c, p, ntiles, tile_rows, c->local_call)) {
    record(c, 5);  // (refine phase = the fused post-scoring kernel; finalize phase empty)
  } else {
    refine(c, p);
    record(c, 5);
    finalize_sum(c, p, ntiles, tile_rows, c->local_call);
  }
  c->summary_packed = c->local_call;
}

__global__ void pack_summary_kernel(const int64_t* __restrict__ checks, const double* __restrict__ result,
                                    const int* __restrict__ missing, HostSummary* out) {
  if (threadIdx.x == 0) {
    out->checks[0] = checks[0];
    out->checks[1] = checks[1];
    out->missing = *missing;
    out->result[0] = result[0];
    out->result[1] = result[1];
    out->result[2] = result[2];
    out->result[3] = result[3];
  }
}

// Reads the (all-reduced) validation word and sum; raises in the reference's order.
double finish(fsil_context* c, double* flagged_out) {
  if (c->phase < 4) fail(FSIL_ERR_INVALID_ARGUMENT, "score must come before finish");
  if (!c->summary_packed) {  // shard mode (words all-reduced since) or an early-out call
    pack_summary_kernel<<<1, 32, 0, c->stream>>>(c->checks.as<int64_t>(), c->result.as<double>(),
                                                 c->counters.as<int>() + 4, c->dsum);
    FSIL_LAUNCHED(c);
  }
  c->summary_packed = false;
  record(c, 6);
  FSIL_CUDA(cudaStreamSynchronize(c->stream));
  const volatile HostSummary* hs = c->hsum;
  if (c->k_spec) {  // the dictionary's count, written by the densify kernels, against the speculated K
    c->k_spec = false;
    const bool over = hs->overflow != 0;
    if (over || hs->count != c->k || (hs->pad && !c->spec_big)) {
      c->spec_missed = true;  // redo the call with the host waiting for the count
      c->spec_block_once = true;
      if (!over) (c->local_call ? c->k_last : c->k_global_last) = hs->count;
      else if (!c->local_call) exchange_grow(c, c->spec_cap_x);  // a rank's dictionary outgrew the exchange
      return 0.0;
    }
  }
  const int64_t checks[2] = {hs->checks[0], hs->checks[1]};
  const double res[4] = {hs->result[0], hs->result[1], hs->result[2], hs->result[3]};
  const int missing = static_cast<int>(hs->missing);
  FSIL_CUDA(cudaGetLastError());
  c->phase = 0;
  if (checks[0] != kNone) {
    const int64_t row = checks[0] / c->d, dim = checks[0] % c->d;
    fail(FSIL_ERR_VALIDATION, "non-finite feature value at point " + std::to_string(row) +
                                  ", dimension " + std::to_string(dim));
  }
  if (c->k < 2)
    fail(FSIL_ERR_VALIDATION, "silhouette undefined for a single cluster: need K >= 2, got K = " +
                                  std::to_string(c->k));
  if (c->metric == FSIL_EUCLID && !c->naive_call)
    fail(FSIL_ERR_VALIDATION,
         "no fast engine for plain euclidean distance (no aggregable decomposition); use the naive "
         "engine");
  if (checks[1] != kNone)
    fail(FSIL_ERR_VALIDATION,
         "cosine distance undefined for zero vector (point " + std::to_string(checks[1]) + ")");
  if (missing) fail(FSIL_ERR_INTERNAL, "a row's label is missing from the dense dictionary");
  c->stats.n = c->n;
  c->stats.d = c->d;
  c->stats.k = c->k;
  c->stats.path = c->score_path;
  c->stats.agg_path = c->agg_path;
  c->stats.flagged_rows = static_cast<int64_t>(res[1]);
  c->stats.exact_rows = static_cast<int64_t>(res[2]);
  c->stats.pair_rows = static_cast<int64_t>(res[3]);
  c->stats.tc_mmas = c->tc_mmas;
  c->stats.tc_threshold = c->tc_thr;
  c->stats.rescored_rows = c->rescored;
  c->stats.kernel_launches = c->launches;
  if (c->timing) {
    float* ms[5] = {&c->stats.ms_densify, &c->stats.ms_aggregate, &c->stats.ms_score,
                    &c->stats.ms_refine, &c->stats.ms_finalize};
    const int from[5] = {0, 1, 3, 4, 5}, to[5] = {1, 2, 4, 5, 6};
    for (int i = 0; i < 5; ++i) FSIL_CUDA(cudaEventElapsedTime(ms[i], c->ev[from[i]], c->ev[to[i]]));
    // ev[7]: recorded by the scoring launcher right before the scoring kernel itself
    c->stats.ms_score_kernel = c->stats.ms_score;
    if (c->ev7_recorded) FSIL_CUDA(cudaEventElapsedTime(&c->stats.ms_score_kernel, c->ev[7], c->ev[4]));
  }
  if (flagged_out) *flagged_out = res[1];
  return res[0] / static_cast<double>(c->n_global);
}

// Dense order = ascending first row (dataset.cpp:41-51).
std::vector<int32_t> order_dictionary(std::vector<std::pair<int64_t, int32_t>>& rows_labels) {
  std::sort(rows_labels.begin(), rows_labels.end());
  std::vector<int32_t> raw(rows_labels.size());
  for (size_t i = 0; i < raw.size(); ++i) raw[i] = rows_labels[i].second;
  return raw;
}

std::vector<std::pair<int64_t, int32_t>> fetch_dictionary(fsil_context* c) {
  std::vector<int32_t> labels(static_cast<size_t>(c->n_distinct));
  std::vector<int64_t> rows(static_cast<size_t>(c->n_distinct));
  if (c->n_distinct > 0) {
    FSIL_CUDA(cudaMemcpyAsync(labels.data(), c->dict_labels.p, labels.size() * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaMemcpyAsync(rows.data(), c->dict_rows.p, rows.size() * sizeof(int64_t),
                              cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
  }
  std::vector<std::pair<int64_t, int32_t>> out(labels.size());
  for (size_t i = 0; i < labels.size(); ++i) out[i] = {rows[i], labels[i]};
  return out;
}

double run_device(fsil_context* c, int metric, const void* dX, bool x64, const int32_t* dlabels, int64_t n,
                  int32_t d, double* ds, int32_t* dnb, int32_t* down, double* da, double* db,
                  int32_t* k_out, int32_t* dense_to_raw) {
  c->launches = 0;
  for (;;) {
    setup(c, metric, dX, x64, dlabels, n, d, 0, n);
    c->local_call = true;
    densify_local(c);  // dictionary ordered on the device (K speculated from the last call)
    record(c, 1);
    c->phase = 2;
    do_aggregate(c);
    do_score(c, ds, dnb, down, da, db);
    if (dense_to_raw && c->k > 0) {  // staged: the caller's buffer holds the true K only
      if (c->k > c->d2r_cap) {
        if (c->d2r_host) FSIL_CUDA(cudaFreeHost(c->d2r_host));
        c->d2r_host = nullptr;
        c->d2r_cap = 0;
        FSIL_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c->d2r_host), c->k * sizeof(int32_t), cudaHostAllocDefault));
        c->d2r_cap = c->k;
      }
      FSIL_CUDA(cudaMemcpyAsync(c->d2r_host, c->dict_sorted_labels, c->k * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                c->stream));
    }
    const double mean = finish(c, nullptr);  // the call's one host sync
    if (c->spec_missed) continue;            // K changed since the last call: once more, unspeculated
    if (dense_to_raw && c->k > 0) std::memcpy(dense_to_raw, c->d2r_host, c->k * sizeof(int32_t));
    if (k_out) *k_out = c->k;
    return mean;
  }
}

template <typename F>
fsil_status guarded(fsil_context* c, F&& f) {
  try {
    f();
    if (c) c->last_error.clear();
    return FSIL_OK;
  } catch (const Error& e) {
    if (c) {
      c->last_error = e.what();
      c->phase = 0;
    }
    return e.status;
  } catch (const std::exception& e) {
    if (c) {
      c->last_error = e.what();
      c->phase = 0;
    }
    return FSIL_ERR_INTERNAL;
  }
}

}  // namespace
}  // namespace fsil

using namespace fsil;

namespace {
thread_local std::string g_create_error;
}

extern "C" {

int fsil_abi_version(void) { return FSIL_ABI_VERSION; }

fsil_status fsil_create(fsil_context** out, int device) {
  if (!out) return FSIL_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  auto* c = new fsil_context();
  const fsil_status st = guarded(c, [&] {
    int count = 0;
    FSIL_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
      fail(FSIL_ERR_CUDA, "no CUDA device " + std::to_string(device) + " (have " + std::to_string(count) + ")");
    cudaDeviceProp prop{};
    FSIL_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(FSIL_ERR_CUDA, std::string("libfsil is built for sm_100a (B200); device is ") + prop.name);
    FSIL_CUDA(cudaSetDevice(device));
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    if (const char* e = std::getenv("FSIL_SPECULATE")) c->speculate = std::string(e) != "0";
    if (const char* e = std::getenv("FSIL_PDL")) c->pdl = std::string(e) != "0";
    if (const char* e = std::getenv("FSIL_DEBUG_SYNC")) c->debug_sync = std::string(e) == "1";
    if (const char* e = std::getenv("FSIL_FUSE_POST")) c->fuse_post = std::string(e) != "0";
    FSIL_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    for (auto& e : c->ev) FSIL_CUDA(cudaEventCreate(&e));
    void* hs = nullptr;
    FSIL_CUDA(cudaHostAlloc(&hs, sizeof(fsil::HostSummary), cudaHostAllocMapped));
    c->hsum = static_cast<fsil::HostSummary*>(hs);
    void* ds = nullptr;
    FSIL_CUDA(cudaHostGetDevicePointer(&ds, hs, 0));
    c->dsum = static_cast<fsil::HostSummary*>(ds);
  });
  if (st != FSIL_OK) {
    g_create_error = c->last_error;  // reachable through fsil_last_error(NULL)
    fsil_destroy(c);
    return st;
  }
  *out = c;
  return FSIL_OK;
}

void fsil_destroy(fsil_context* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  fsil::DevBuf* bufs[] = {&c->ht_keys, &c->ht_vals, &c->ht_dense, &c->dict_labels, &c->dict_rows,
                          &c->counters, &c->dict_sorted, &c->dense, &c->stats_buf, &c->checks, &c->partials,
                          &c->sort_tmp, &c->sort_keys, &c->sort_vals, &c->iota, &c->seg_start,
                          &c->piece_start, &c->mu32, &c->p32, &c->nk, &c->bound, &c->s_tmp,
                          &c->tile_sum, &c->tile_flag, &c->flag_rows, &c->flag_count, &c->result,
                          &c->group_sum, &c->xmax, &c->tc_b, &c->nb_tmp, &c->pair_rows, &c->pair_count, &c->thr_nn, &c->thr_t, &c->cand_rows, &c->a_scratch, &c->x32, &c->xbuf, &c->xt_keys, &c->xt_vals, &c->xt_dense, &c->hX, &c->hL, &c->o_s, &c->o_nb, &c->o_own, &c->o_a,
                          &c->o_b, &c->refine_part, &c->refine_cnt, &c->sub_x, &c->sub_i, &c->xi_rows};
  for (auto* b : bufs) b->release();
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->hsum) cudaFreeHost(c->hsum);
  if (c->d2r_host) cudaFreeHost(c->d2r_host);
  delete c;
}

const char* fsil_last_error(const fsil_context* c) {
  return c ? c->last_error.c_str() : g_create_error.c_str();
}

fsil_status fsil_set_stream(fsil_context* c, void* stream) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (stream) {
      if (c->own_stream && c->stream) FSIL_CUDA(cudaStreamDestroy(c->stream));
      c->stream = static_cast<cudaStream_t>(stream);
      c->own_stream = false;
    } else if (!c->own_stream) {
      FSIL_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
  });
}

fsil_status fsil_set_path(fsil_context* c, int path) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  if (path < FSIL_PATH_AUTO || path > FSIL_PATH_FP64) {
    c->last_error = "unknown scoring path";
    return FSIL_ERR_INVALID_ARGUMENT;
  }
  c->path = path;
  return FSIL_OK;
}

fsil_status fsil_set_timing(fsil_context* c, int enabled) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  c->timing = enabled != 0;
  return FSIL_OK;
}

fsil_status fsil_get_stats(const fsil_context* c, fsil_stats* out) {
  if (!c || !out) return FSIL_ERR_INVALID_ARGUMENT;
  *out = c->stats;
  return FSIL_OK;
}

fsil_status fsil_silhouette_device(fsil_context* c, int metric, const float* dX,
                                   const int32_t* dlabels, int64_t n, int32_t d, double* ds,
                                   int32_t* dnb, int32_t* down, double* da, double* db,
                                   double* mean, int32_t* k_out, int32_t* dense_to_raw) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    const double m = run_device(c, metric, dX, false, dlabels, n, d, ds, dnb, down, da, db, k_out, dense_to_raw);
    if (mean) *mean = m;
  });
}
fsil_status fsil_silhouette_device_f64(fsil_context* c, int metric, const double* dX, const int32_t* dlabels,
                                       int64_t n, int32_t d, double* ds, int32_t* dnb, int32_t* down, double* da,
                                       double* db, double* mean, int32_t* k_out, int32_t* dense_to_raw) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    const double m = run_device(c, metric, dX, true, dlabels, n, d, ds, dnb, down, da, db, k_out, dense_to_raw);
    if (mean) *mean = m;
  });
}

}  // extern "C"

namespace {
// Host buffers: copy X (fp32 or fp64) and labels to HBM, run, copy results back.
template <typename T>
fsil_status host_call(fsil_context* c, int metric, const T* X, const int32_t* labels, int64_t n, int32_t d,
                      double* s, int32_t* neighbour, int32_t* own, double* a, double* b, double* mean,
                      int32_t* k_out, int32_t* dense_to_raw, bool naive = false) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  struct NaiveScope {  // the engine flag lasts for this call only
    fsil_context* c;
    ~NaiveScope() { c->naive_call = false; }
  } scope{c};
  c->naive_call = naive;
  return guarded(c, [&] {
    check_metric(metric);
    check_shape(n, d);
    if (!X || !labels) fail(FSIL_ERR_INVALID_ARGUMENT, "null input pointer");
    FSIL_CUDA(cudaSetDevice(c->device));
    const size_t xb = static_cast<size_t>(n) * d * sizeof(T);
    c->hX.ensure(xb);
    c->hL.ensure(n * sizeof(int32_t));
    FSIL_CUDA(cudaMemcpyAsync(c->hX.p, X, xb, cudaMemcpyHostToDevice, c->stream));
    FSIL_CUDA(cudaMemcpyAsync(c->hL.p, labels, n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
    double* ds = nullptr;
    int32_t *dnb = nullptr, *down = nullptr;
    double *da = nullptr, *db = nullptr;
    if (s) { c->o_s.ensure(n * sizeof(double)); ds = c->o_s.as<double>(); }
    if (neighbour) { c->o_nb.ensure(n * sizeof(int32_t)); dnb = c->o_nb.as<int32_t>(); }
    if (own) { c->o_own.ensure(n * sizeof(int32_t)); down = c->o_own.as<int32_t>(); }
    if (a) { c->o_a.ensure(n * sizeof(double)); da = c->o_a.as<double>(); }
    if (b) { c->o_b.ensure(n * sizeof(double)); db = c->o_b.as<double>(); }
    const double m = run_device(c, metric, c->hX.p, sizeof(T) == 8, c->hL.as<int32_t>(), n, d, ds, dnb, down, da,
                                db, k_out, dense_to_raw);
    if (s) FSIL_CUDA(cudaMemcpyAsync(s, ds, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (neighbour) FSIL_CUDA(cudaMemcpyAsync(neighbour, dnb, n * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    if (own) FSIL_CUDA(cudaMemcpyAsync(own, down, n * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    if (a) FSIL_CUDA(cudaMemcpyAsync(a, da, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (b) FSIL_CUDA(cudaMemcpyAsync(b, db, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    if (mean) *mean = m;
  });
}
}  // namespace

extern "C" {

fsil_status fsil_silhouette(fsil_context* c, int metric, const float* X, const int32_t* labels, int64_t n,
                            int32_t d, double* s, int32_t* neighbour, int32_t* own, double* a, double* b,
                            double* mean, int32_t* k_out, int32_t* dense_to_raw) {
  return host_call(c, metric, X, labels, n, d, s, neighbour, own, a, b, mean, k_out, dense_to_raw);
}
fsil_status fsil_silhouette_f64(fsil_context* c, int metric, const double* X, const int32_t* labels, int64_t n,
                                int32_t d, double* s, int32_t* neighbour, int32_t* own, double* a, double* b,
                                double* mean, int32_t* k_out, int32_t* dense_to_raw) {
  return host_call(c, metric, X, labels, n, d, s, neighbour, own, a, b, mean, k_out, dense_to_raw);
}
fsil_status fsil_silhouette_naive(fsil_context* c, int metric, const double* X, const int32_t* labels, int64_t n,
                                  int32_t d, double* s, int32_t* neighbour, int32_t* own, double* a, double* b,
                                  double* mean, int32_t* k_out, int32_t* dense_to_raw) {
  return host_call(c, metric, X, labels, n, d, s, neighbour, own, a, b, mean, k_out, dense_to_raw, true);
}
fsil_status fsil_shard_begin(fsil_context* c, int metric, const float* dX, const int32_t* dlabels,
                             int64_t n_local, int32_t d, int64_t row_offset, int64_t n_global,
                             int64_t* n_distinct) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    begin(c, metric, dX, false, dlabels, n_local, d, row_offset, n_global);
    if (n_distinct) *n_distinct = c->n_distinct;
  });
}
fsil_status fsil_shard_begin_f64(fsil_context* c, int metric, const double* dX, const int32_t* dlabels,
                                 int64_t n_local, int32_t d, int64_t row_offset, int64_t n_global,
                                 int64_t* n_distinct) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    begin(c, metric, dX, true, dlabels, n_local, d, row_offset, n_global);
    if (n_distinct) *n_distinct = c->n_distinct;
  });
}

fsil_status fsil_shard_begin_device(fsil_context* c, int metric, const void* dX, int xtype, const int32_t* dlabels,
                                    int64_t n_local, int32_t d, int64_t row_offset, int64_t n_global,
                                    int64_t** d_entries, int64_t* capacity) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (xtype != 0 && xtype != 1) fail(FSIL_ERR_INVALID_ARGUMENT, "xtype: 0 (fp32) or 1 (fp64)");
    c->launches = 0;
    setup(c, metric, dX, xtype == 1, dlabels, n_local, d, row_offset, n_global);
    c->local_call = false;
    // the same capacity on every rank: from the previous call's global K (identical everywhere)
    int64_t cap_x = 64;
    while (cap_x < 2 * c->k_global_last + 2) cap_x *= 2;
    int64_t* buf = densify_exchange_begin(c, cap_x);
    c->phase = 1;
    if (d_entries) *d_entries = buf;
    if (capacity) *capacity = cap_x;
  });
}
fsil_status fsil_shard_set_dictionary_device(fsil_context* c, const int64_t* d_gathered, int32_t nranks,
                                             int64_t capacity) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (c->phase < 1) fail(FSIL_ERR_INVALID_ARGUMENT, "fsil_shard_begin_device must come first");
    if (!d_gathered || nranks < 1 || capacity < 2) fail(FSIL_ERR_INVALID_ARGUMENT, "bad exchange buffer");
    densify_exchange_set(c, d_gathered, nranks, capacity);
    c->k_global_last = c->k;
    record(c, 1);
    c->phase = 2;
  });
}

fsil_status fsil_shard_get_dictionary(fsil_context* c, int32_t* raw_labels, int64_t* first_rows) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    if (c->phase < 1) fail(FSIL_ERR_INVALID_ARGUMENT, "fsil_shard_begin must come first");
    auto dict = fetch_dictionary(c);
    std::sort(dict.begin(), dict.end());
    for (size_t i = 0; i < dict.size(); ++i) {
      if (raw_labels) raw_labels[i] = dict[i].second;
      if (first_rows) first_rows[i] = dict[i].first;
    }
  });
}

fsil_status fsil_shard_set_dictionary(fsil_context* c, const int32_t* raw, int32_t k) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] { set_dictionary(c, raw, k); });
}

fsil_status fsil_shard_aggregate(fsil_context* c, double** d_stats, int64_t* stats_len,
                                 int64_t** d_checks) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    do_aggregate(c);
    const int m = c->metric == FSIL_EUCLID ? FSIL_SQEUCLID : c->metric;
    if (d_stats) *d_stats = c->stats_buf.as<double>();
    if (stats_len) *stats_len = StatsLayout{m, c->k, c->d}.len();
    if (d_checks) *d_checks = c->checks.as<int64_t>();
  });
}

fsil_status fsil_shard_score(fsil_context* c, double* ds, int32_t* dnb, int32_t* down, double* da,
                             double* db, double** d_partial) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    do_score(c, ds, dnb, down, da, db);
    if (d_partial) *d_partial = c->result.as<double>();
  });
}

fsil_status fsil_shard_finish(fsil_context* c, double* mean) {
  if (!c) return FSIL_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    const double m = finish(c, nullptr);
    if (c->spec_missed)
      fail(FSIL_AGAIN, "the global number of clusters changed since the previous call: repeat the protocol "
                       "from fsil_shard_begin_device");
    if (mean) *mean = m;
  });
}

fsil_status fsil_plan_shards(int64_t n, int32_t requested, int64_t* ranges, int32_t* num_shards) {
  if (n < 1 || requested < 1 || !ranges) return FSIL_ERR_INVALID_ARGUMENT;
  const int64_t w = std::min<int64_t>(requested, n);
  const int64_t base = n / w, extra = n % w;
  int64_t begin = 0;
  for (int64_t s = 0; s < w; ++s) {
    const int64_t size = base + (s < extra ? 1 : 0);
    ranges[2 * s] = begin;
    ranges[2 * s + 1] = begin + size;
    begin += size;
  }
  if (num_shards) *num_shards = static_cast<int32_t>(w);
  return FSIL_OK;
}

fsil_status fsil_assemble_score(double a, double b, double* s) {
  if (!s || a < 0.0 || b < 0.0) return FSIL_ERR_INVALID_ARGUMENT;
  *s = (a == 0.0 && b == 0.0) ? 0.0 : (a <= b ? 1.0 - a / b : b / a - 1.0);
  return FSIL_OK;
}

}  // extern "C"
