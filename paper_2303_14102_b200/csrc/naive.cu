// naive.cu -- the Theta(N^2 D) engine on the GPU: every pairwise distance
// in fp64, for the reference's compare contract and the metric the linear engine cannot
// serve (plain Euclidean).
//
// Follows naive_silhouette (naive.cpp:30-71) and pairwise_distance (naive.cpp:12-28):
// per row i, sums[k] += d(x_i, x_j) over j != i in ascending j; a = sums[own]/(n_own-1)
// (0 for a singleton), b = min over k != own of sums[k]/n_k (strict <, ascending k),
// s by make_point_score.  Distances: squared norm of the difference, its square root,
// or 1 - dot/(|p||q|).  One thread per row (128 rows per block); j tiles of 64 rows are
// staged in shared memory; the per-row cluster sums live in shared memory laid out
// [k][thread], so a warp's updates for one j (same label) are conflict free.
#include <algorithm>

#include "score_common.cuh"

namespace fsil {
namespace {

constexpr int kRows = 128, kTile = 64;

template <int METRIC>
__global__ void __launch_bounds__(kRows) naive_kernel(const double* __restrict__ X, const int32_t* __restrict__ dense,
                                                      const double* __restrict__ counts, int64_t n, int d, int k,
                                                      double* s_out, int32_t* nb_out, int32_t* own_out, double* a_out,
                                                      double* b_out, double* tile_sum, int32_t* tile_flag) {
  extern __shared__ double sm[];
  double* acc = sm;                    // [k][kRows]
  double* xj = acc + k * kRows;        // [kTile][d]
  double* nj = xj + kTile * d;         // [kTile] norms (cosine)
  int* lj = reinterpret_cast<int*>(nj + kTile);  // [kTile] labels
  const int tid = threadIdx.x;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kRows + tid;
  const bool valid = i < n;
  for (int c = 0; c < k; ++c) acc[c * kRows + tid] = 0.0;
  const double* xi = X + (valid ? i : 0) * d;
  double ni = 0.0;
  if (METRIC == FSIL_COSINE) {
    for (int l = 0; l < d; ++l) ni = fma(xi[l], xi[l], ni);
    ni = sqrt(ni);
  }
  for (int64_t j0 = 0; j0 < n; j0 += kTile) {
    const int cnt = static_cast<int>(n - j0 < kTile ? n - j0 : kTile);
    __syncthreads();
    for (int e = tid; e < cnt * d; e += kRows) xj[e] = X[j0 * d + e];
    for (int e = tid; e < cnt; e += kRows) lj[e] = dense[j0 + e];
    __syncthreads();
    if (METRIC == FSIL_COSINE) {
      for (int e = tid; e < cnt; e += kRows) {
        double q = 0.0;
        for (int l = 0; l < d; ++l) q = fma(xj[e * d + l], xj[e * d + l], q);
        nj[e] = sqrt(q);
      }
      __syncthreads();
    }
    for (int jj = 0; jj < cnt; ++jj) {
      const int64_t j = j0 + jj;
      const double* q = xj + jj * d;
      double dist;
      if (METRIC == FSIL_COSINE) {
        double dot = 0.0;
        for (int l = 0; l < d; ++l) dot = fma(xi[l], q[l], dot);
        dist = 1.0 - dot / (ni * nj[jj]);
      } else {
        double ss = 0.0;
        for (int l = 0; l < d; ++l) {
          const double t = xi[l] - q[l];
          ss = fma(t, t, ss);
        }
        dist = METRIC == FSIL_EUCLID ? sqrt(ss) : ss;
      }
      if (valid && j != i) acc[lj[jj] * kRows + tid] += dist;
    }
  }
  double s = 0.0;
  if (valid) {
    const int own = dense[i];
    const double n_own = counts[own];
    const bool singleton = n_own == 1.0;
    const double a = singleton ? 0.0 : acc[own * kRows + tid] / (n_own - 1.0);
    double best = INFINITY;
    int nb = -1;
    for (int c = 0; c < k; ++c) {
      if (c == own) continue;
      const double mean = acc[c * kRows + tid] / counts[c];
      if (mean < best) {
        best = mean;
        nb = c;
      }
    }
    s = singleton ? 0.0 : assemble_score(a, best);
    s_out[i] = s;
    if (nb_out) nb_out[i] = nb;
    if (own_out) own_out[i] = own;
    if (a_out) a_out[i] = a;
    if (b_out) b_out[i] = best;
  }
  // per-block partial of the fixed-order mean (tile = kRows rows)
  __shared__ double red[kRows / 32];
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kRows / 32; ++w) t += red[w];
    tile_sum[blockIdx.x] = t;
    tile_flag[blockIdx.x] = 0;
  }
}

}  // namespace

int64_t naive_tiles(int64_t n, int* tile_rows) {
  *tile_rows = kRows;
  return (n + kRows - 1) / kRows;
}

void score_naive(fsil_context* c, const ScoreParams& p) {
  if (!c->X64) fail(FSIL_ERR_INTERNAL, "naive engine: fp64 features expected");
  const size_t smem = (static_cast<size_t>(c->k) * kRows + static_cast<size_t>(kTile) * c->d + kTile) * sizeof(double) +
                      kTile * sizeof(int);
  if (smem > c->smem_optin)
    fail(FSIL_ERR_INVALID_ARGUMENT, "naive engine: K x 128 + 64 x D doubles exceed shared memory (K=" +
                                        std::to_string(c->k) + ", D=" + std::to_string(c->d) + ")");
  const unsigned grid = static_cast<unsigned>((c->n + kRows - 1) / kRows);
  const double* counts = p.stats;  // StatsLayout: [count K] first
#define FSIL_NAIVE(M)                                                                                       \
  {                                                                                                         \
    FSIL_CUDA(cudaFuncSetAttribute(naive_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    naive_kernel<M><<<grid, kRows, smem, c->stream>>>(c->X64, p.dense, counts, c->n, c->d, c->k, p.s, p.nb,     \
                                                      p.own, p.a, p.b, p.tile_sum, p.tile_flag);             \
  }
  if (c->metric == FSIL_COSINE) FSIL_NAIVE(FSIL_COSINE)
  else if (c->metric == FSIL_EUCLID) FSIL_NAIVE(FSIL_EUCLID)
  else FSIL_NAIVE(FSIL_SQEUCLID)
#undef FSIL_NAIVE
  FSIL_LAUNCHED(c);
}

}  // namespace fsil
