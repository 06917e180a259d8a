// aggregate.cu -- K1: label-segmented fp64 cluster statistics.
//
// Replaces aggregate_cluster_stats / Policy::partial / Policy::merge
// (engine.hpp:50-80; squared_euclidean.cpp:37-63; cosine.cpp:39-69):
//   sqeuclid: N_k, Psi_k = sum ||x||^2, Y_k = sum x
//   cosine  : N_k, Omega_k = sum x / ||x||   (zero-norm rows rejected, cos.cpp:119-123)
// fused with the dataset validation the reference does before it (finite
// values, dataset.cpp:35-37).  Two deterministic device paths:
//   1. warp-private shared-memory copies when K*(D+2) is small (C1, C2): each
//      row-slot owns a private fp64 copy, rows are assigned to slots by a fixed
//      rule, copies and block partials are folded in fixed order;
//   2. label-sorted segments for large K*D (C3..C5): a stable radix sort of
//      (dense label, row) pairs makes every cluster a contiguous run of row ids;
//      warps reduce fixed-size pieces of a run in registers (fp64) and a fold
//      kernel sums the pieces of each cluster in order.
// Both read X exactly once with coalesced 128-bit loads; neither uses
// floating-point atomics, so results are bit-identical run to run.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "device_util.cuh"
#include "fsil_internal.cuh"

namespace fsil {
namespace {

constexpr int kPieceRows = 2048;

// ---------------------------------------------------------------- path 1 ----
// Lanes of a warp are split into RPW row sub-groups of LPR lanes; each lane
// covers CPL chunks of VEC floats of the row.  Copy index = warp*RPW + sub.
// Within a copy the cluster sums are stored "chunk-transposed" (element l at
// (l%VEC)*nchunks + l/VEC) so that a sub-group's read-modify-writes hit
// consecutive doubles (bank-conflict free).  U rows per slot are loaded ahead.
template <bool COS, int VEC, int CPL>
__global__ void __launch_bounds__(256) agg_private_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ dense, int64_t n, int d,
    int64_t row_offset, int k, int lpr, double* __restrict__ partials, int64_t* checks,
    float* xmax) {
  constexpr int U = 4;
  float amax = 0.f;
  extern __shared__ double sm[];
  const int S = COS ? k * (d + 1) : k * (d + 2);
  const int sums_off = COS ? k : 2 * k;
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rpw = 32 / lpr;
  const int sub = lane / lpr, li = lane % lpr;
  const int copies = warps * rpw;
  for (int j = threadIdx.x; j < copies * S; j += blockDim.x) sm[j] = 0.0;
  __syncthreads();
  double* my = sm + (warp * rpw + sub) * S;
  const int64_t G = static_cast<int64_t>(gridDim.x) * copies;
  const int nchunks = (d + VEC - 1) / VEC;
  const int64_t wbase = (static_cast<int64_t>(blockIdx.x) * warps + warp) * rpw;
  for (int64_t base = wbase; base < n; base += U * G) {
    float v[U][CPL][VEC];
    int lab[U];
    bool valid[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = base + sub + u * G;
      valid[u] = r < n;
      lab[u] = valid[u] ? __ldg(dense + r) : 0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int ch = li + c * lpr;
        if constexpr (VEC == 4) {
          float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
          if (valid[u] && ch < nchunks) t = ldg_stream(reinterpret_cast<const float4*>(X + r * d) + ch);
          v[u][c][0] = t.x; v[u][c][1] = t.y; v[u][c][2] = t.z; v[u][c][3] = t.w;
        } else {
          v[u][c][0] = (valid[u] && ch < nchunks) ? __ldg(X + r * d + ch) : 0.f;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = base + sub + u * G;
      double ss = 0.0;
      bool finite = true;
#pragma unroll
      for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const double x = v[u][c][e];
          ss = fma(x, x, ss);
          finite = finite && isfinite(v[u][c][e]);
          amax = fmaxf(amax, fabsf(v[u][c][e]));
        }
      if (!finite) {
#pragma unroll
        for (int c = 0; c < CPL; ++c)
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const int l = (li + c * lpr) * VEC + e;
            if (l < d && !isfinite(v[u][c][e])) atomic_min_i64(checks, (row_offset + r) * d + l);
          }
      }
      for (int off = lpr >> 1; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off, lpr);
      if (!valid[u]) continue;
      double scale = 1.0;
      if (COS) {
        if (ss == 0.0) {
          if (li == 0) atomic_min_i64(checks + 1, row_offset + r);
          continue;
        }
        scale = 1.0 / sqrt(ss);
      }
      if (li == 0) {
        my[lab[u]] += 1.0;
        if (!COS) my[k + lab[u]] += ss;
      }
      double* ys = my + sums_off + static_cast<int64_t>(lab[u]) * d;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int ch = li + c * lpr;
        if (ch < nchunks) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const double x = COS ? static_cast<double>(v[u][c][e]) * scale : static_cast<double>(v[u][c][e]);
            ys[e * nchunks + ch] += x;
          }
        }
      }
    }
  }
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  if (lane == 0 && amax > 0.f) atomic_max_nonneg_f32(xmax, amax);
  __syncthreads();
  for (int j = threadIdx.x; j < S; j += blockDim.x) {
    int src = j;
    if (j >= sums_off) {  // undo the chunk transpose
      const int t = j - sums_off, kk = t / d, l = t % d;
      src = sums_off + kk * d + (l % VEC) * nchunks + l / VEC;
    }
    double acc = 0.0;
    for (int c = 0; c < copies; ++c) acc += sm[c * S + src];
    partials[static_cast<int64_t>(blockIdx.x) * S + j] = acc;
  }
}

// Sum of block partials per element: 8 fixed strided chains + fixed tree.
__global__ void __launch_bounds__(256) fold_partials_kernel(const double* __restrict__ partials,
                                                            int nblocks, int64_t S,
                                                            double* __restrict__ stats) {
  __shared__ double sm[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  double acc = 0.0;
  if (j < S)
    for (int b = ty; b < nblocks; b += 8) acc += partials[b * S + j];
  sm[ty][tx] = acc;
  __syncthreads();
  if (ty == 0 && j < S) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sm[w][tx];
    stats[j] = t;
  }
}

// ---------------------------------------------------------------- path 2 ----
__global__ void iota_kernel(int32_t* v, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<int32_t>(i);
}

__global__ void segment_bounds_kernel(const int32_t* __restrict__ keys, int64_t n,
                                      int64_t* seg_begin, int64_t* seg_end) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t key = keys[i];
  if (i == 0 || keys[i - 1] != key) seg_begin[key] = i;
  if (i == n - 1 || keys[i + 1] != key) seg_end[key] = i + 1;
}

__global__ void pieces_per_cluster_kernel(const int64_t* seg_begin, const int64_t* seg_end, int k,
                                          int64_t* ppc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > k) return;
  ppc[j] = j < k ? (seg_end[j] - seg_begin[j] + kPieceRows - 1) / kPieceRows : 0;
}

// One warp per piece of <= kPieceRows rows of one cluster, rows gathered via
// the sorted row ids.  Lanes: RPW row sub-groups of LPR lanes; CPL chunks of
// VEC floats per lane.  Piece partial layout: [count][psi][sums d] (psi only
// for sqeuclid).
template <bool COS, int VEC, int CPL>
__global__ void __launch_bounds__(256) agg_piece_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ rows, int64_t n, int d,
    int64_t row_offset, int k, int lpr, const int64_t* __restrict__ seg_begin,
    const int64_t* __restrict__ seg_end, const int64_t* __restrict__ piece_start,
    double* __restrict__ piece_out, int64_t* checks, float* xmax) {
  const int64_t p = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t total = piece_start[k];
  if (p >= total) return;
  // cluster owning piece p: largest c with piece_start[c] <= p
  int lo = 0, hi = k - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (piece_start[mid] <= p) lo = mid;
    else hi = mid - 1;
  }
  const int c = lo;
  const int64_t b0 = seg_begin[c] + (p - piece_start[c]) * kPieceRows;
  const int64_t b1 = min(seg_end[c], b0 + kPieceRows);
  const int rpw = 32 / lpr;
  const int sub = lane / lpr, li = lane % lpr;
  const int nchunks = (d + VEC - 1) / VEC;
  double acc[CPL][VEC];
#pragma unroll
  for (int q = 0; q < CPL; ++q)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[q][e] = 0.0;
  double psi = 0.0, cnt = 0.0;
  float amax = 0.f;
  for (int64_t base = b0; base < b1; base += rpw) {
    const int64_t pos = base + sub;  // warp-uniform trip count
    const bool valid = pos < b1;
    const int64_t r = valid ? rows[pos] : 0;
    float v[CPL][VEC];
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int ch = li + q * lpr;
      if constexpr (VEC == 4) {
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid && ch < nchunks) t = ldg_stream(reinterpret_cast<const float4*>(X + r * d) + ch);
        v[q][0] = t.x; v[q][1] = t.y; v[q][2] = t.z; v[q][3] = t.w;
      } else {
        v[q][0] = (valid && ch < nchunks) ? __ldg(X + r * d + ch) : 0.f;
      }
    }
    double ss = 0.0;
    bool finite = true;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const double x = v[q][e];
        ss += x * x;
        finite = finite && isfinite(v[q][e]);
        amax = fmaxf(amax, fabsf(v[q][e]));
      }
    if (!finite) {
#pragma unroll
      for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const int l = (li + q * lpr) * VEC + e;
          if (l < d && !isfinite(v[q][e])) atomic_min_i64(checks, (row_offset + r) * d + l);
        }
    }
    double scale = 1.0;
    if (COS) {
      for (int off = lpr >> 1; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off, lpr);
      if (!valid) continue;
      if (ss == 0.0) {
        if (li == 0) atomic_min_i64(checks + 1, row_offset + r);
        continue;
      }
      scale = 1.0 / sqrt(ss);
    } else {
      if (!valid) continue;
      psi += ss;  // per-lane partial of sum ||x||^2, reduced below
    }
    cnt += 1.0;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        acc[q][e] += COS ? static_cast<double>(v[q][e]) * scale : static_cast<double>(v[q][e]);
  }
  // Combine row sub-groups (fixed xor order) so sub-group 0 holds the piece sums.
  for (int off = 16; off >= lpr; off >>= 1) {
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[q][e] += __shfl_xor_sync(0xffffffffu, acc[q][e], off);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  if (!COS)
    for (int off = 16; off > 0; off >>= 1) psi += __shfl_xor_sync(0xffffffffu, psi, off);
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  if (lane == 0 && amax > 0.f) atomic_max_nonneg_f32(xmax, amax);
  const int S1 = COS ? d + 1 : d + 2;
  double* out = piece_out + p * S1;
  if (lane == 0) {
    out[0] = cnt;
    if (!COS) out[1] = psi;
  }
  if (sub == 0) {
    double* sums = out + (COS ? 1 : 2);
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const int l = (li + q * lpr) * VEC + e;
        if (l < d) sums[l] = acc[q][e];
      }
  }
}

__global__ void fold_pieces_kernel(const double* __restrict__ piece_out,
                                   const int64_t* __restrict__ piece_start, int k, int d, bool cos,
                                   double* __restrict__ stats) {
  const int S1 = cos ? d + 1 : d + 2;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(k) * S1) return;
  const int c = static_cast<int>(t / S1), j = static_cast<int>(t % S1);
  double acc = 0.0;
  for (int64_t p = piece_start[c]; p < piece_start[c + 1]; ++p) acc += piece_out[p * S1 + j];
  if (j == 0) stats[c] = acc;
  else if (!cos && j == 1) stats[k + c] = acc;
  else stats[(cos ? k : 2 * k) + static_cast<int64_t>(c) * d + (j - (cos ? 1 : 2))] = acc;
}

// ---------------------------------------------------------------- derive ----
// Per-cluster constants of the scoring pass (fp32 operand copies + bounds).
__global__ void derive_kernel(const double* __restrict__ stats, int k, int d, int dp, bool cos,
                              float* mu32, float* p32, double* nk, float* bound) {
  const int c = blockIdx.x;
  const double cnt = stats[c];
  const double n = cnt > 0.0 ? cnt : 1.0;
  const double* sums = stats + (cos ? k : 2 * k) + static_cast<int64_t>(c) * d;
  double sq = 0.0;
  float amax = 0.f;
  for (int l = threadIdx.x; l < dp; l += blockDim.x) {
    const double m = l < d ? sums[l] / n : 0.0;
    mu32[static_cast<int64_t>(c) * dp + l] = static_cast<float>(m);
    sq += m * m;
    amax = fmaxf(amax, __double2float_ru(fabs(m)));
  }
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  if ((threadIdx.x & 31) == 0 && amax > 0.f) atomic_max_nonneg_f32(bound + 2, amax);
  __shared__ double red[32];
  for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) tot += red[w];
    nk[c] = cnt;
    atomic_max_nonneg_f32(bound + 0, __double2float_ru(sqrt(tot) * (1.0 + 1e-12)));
    if (!cos) {
      const double p = stats[k + c] / n;
      p32[c] = static_cast<float>(p);
      atomic_max_nonneg_f32(bound + 1, __double2float_ru(fabs(p) * (1.0 + 1e-12)));
    }
  }
}

int pick_lpr(int d, int vec) {
  const int chunks = (d + vec - 1) / vec;
  int lpr = 1;
  while (lpr < chunks && lpr < 32) lpr <<= 1;
  return lpr;
}

template <bool COS>
void launch_private(fsil_context* c, int vec, int cpl, int grid, int threads, int lpr,
                    size_t smem, double* partials, int64_t* checks) {
#define FSIL_AGG_PRIV(V, C)                                                                      \
  if (vec == V && cpl == C) {                                                                    \
    auto kern = agg_private_kernel<COS, V, C>;                                                   \
    FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    kern<<<grid, threads, smem, c->stream>>>(c->X, c->dense.as<int32_t>(), c->n, c->d,          \
                                             c->row_offset, c->k, lpr, partials, checks,         \
                                             c->xmax.as<float>());                               \
    FSIL_LAUNCHED(c);                                                                            \
    return;                                                                                      \
  }
  FSIL_AGG_PRIV(4, 1) FSIL_AGG_PRIV(4, 2) FSIL_AGG_PRIV(4, 4)
  FSIL_AGG_PRIV(1, 1) FSIL_AGG_PRIV(1, 2) FSIL_AGG_PRIV(1, 4)
#undef FSIL_AGG_PRIV
  fail(FSIL_ERR_INTERNAL, "no private aggregation kernel for this shape");
}

template <bool COS>
void launch_pieces(fsil_context* c, int vec, int cpl, int64_t max_pieces, int lpr,
                   const int32_t* rows, int64_t* seg_begin, int64_t* seg_end,
                   int64_t* piece_start, double* piece_out, int64_t* checks) {
  const unsigned grid = static_cast<unsigned>((max_pieces * 32 + 255) / 256);
#define FSIL_AGG_PIECE(V, C)                                                                     \
  if (vec == V && cpl == C) {                                                                    \
    agg_piece_kernel<COS, V, C><<<grid, 256, 0, c->stream>>>(                                    \
        c->X, rows, c->n, c->d, c->row_offset, c->k, lpr, seg_begin, seg_end, piece_start,       \
        piece_out, checks, c->xmax.as<float>());                                                 \
    FSIL_LAUNCHED(c);                                                                            \
    return;                                                                                      \
  }
  FSIL_AGG_PIECE(4, 1) FSIL_AGG_PIECE(4, 2) FSIL_AGG_PIECE(4, 4) FSIL_AGG_PIECE(4, 8)
  FSIL_AGG_PIECE(1, 1) FSIL_AGG_PIECE(1, 2) FSIL_AGG_PIECE(1, 4) FSIL_AGG_PIECE(1, 8)
  FSIL_AGG_PIECE(1, 16) FSIL_AGG_PIECE(1, 32)
#undef FSIL_AGG_PIECE
  fail(FSIL_ERR_INTERNAL, "no piece aggregation kernel for this shape");
}

}  // namespace

void aggregate(fsil_context* c) {
  const bool cos = c->metric == FSIL_COSINE;
  const StatsLayout L{c->metric, c->k, c->d};
  const int64_t S = L.len();
  c->stats_buf.ensure(S * sizeof(double));
  c->checks.ensure(2 * sizeof(int64_t));
  double* stats = c->stats_buf.as<double>();
  int64_t* checks = c->checks.as<int64_t>();
  const int64_t none[2] = {kNone, kNone};
  FSIL_CUDA(cudaMemcpyAsync(checks, none, sizeof(none), cudaMemcpyHostToDevice, c->stream));
  FSIL_CUDA(cudaMemsetAsync(stats, 0, S * sizeof(double), c->stream));
  c->xmax.ensure(sizeof(float));
  FSIL_CUDA(cudaMemsetAsync(c->xmax.p, 0, sizeof(float), c->stream));
  if (c->n == 0) {
    c->agg_path = 0;
    return;
  }
  const int vec = (c->d % 4 == 0) ? 4 : 1;
  const int lpr = pick_lpr(c->d, vec);
  const int chunks = (c->d + vec - 1) / vec;
  const int cpl = (chunks + lpr - 1) / lpr;
  const int rpw = 32 / lpr;

  // Path 1: warp-private shared-memory copies; needs >= 8 resident warps/SM.
  const size_t budget = c->smem_optin ? c->smem_optin : 227 * 1024;
  int warps = 8;
  size_t smem = 0;
  for (; warps >= 1; warps >>= 1) {
    smem = static_cast<size_t>(warps) * rpw * S * sizeof(double);
    if (smem <= budget) break;
  }
  const int blocks_per_sm = warps >= 1 && smem > 0 ? static_cast<int>(budget / smem) : 0;
  const bool private_ok = warps >= 1 && cpl <= 4 && blocks_per_sm >= 1 &&
                          warps * std::min(blocks_per_sm, 8) >= 8;
  if (private_ok) {
    c->agg_path = 1;
    const int per_sm = std::min(blocks_per_sm, 64 / warps);
    const int64_t rows_per_block = static_cast<int64_t>(warps) * rpw * 8;
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>((c->n + rows_per_block - 1) / rows_per_block,
                             static_cast<int64_t>(c->num_sms) * per_sm)));
    c->partials.ensure(static_cast<size_t>(grid) * S * sizeof(double));
    const int cpl_t = cpl <= 1 ? 1 : cpl <= 2 ? 2 : 4;
    if (cos)
      launch_private<true>(c, vec, cpl_t, grid, warps * 32, lpr, smem, c->partials.as<double>(), checks);
    else
      launch_private<false>(c, vec, cpl_t, grid, warps * 32, lpr, smem, c->partials.as<double>(), checks);
    fold_partials_kernel<<<static_cast<unsigned>((S + 31) / 32), 256, 0, c->stream>>>(
        c->partials.as<double>(), grid, S, stats);
    FSIL_LAUNCHED(c);
    return;
  }

  // Path 2: label-sorted segments.
  if (c->n >= (int64_t(1) << 31)) fail(FSIL_ERR_INVALID_ARGUMENT, "shard too large for the sorted aggregation path (2^31 rows)");
  const int cpl_max = vec == 4 ? 8 : 32;
  if (cpl > cpl_max)
    fail(FSIL_ERR_INVALID_ARGUMENT, "feature dimension too large for this build (D <= 1024)");
  c->agg_path = 2;
  const int n32 = static_cast<int>(c->n);
  c->iota.ensure(c->n * sizeof(int32_t));
  c->sort_keys.ensure(c->n * sizeof(int32_t));
  c->sort_vals.ensure(c->n * sizeof(int32_t));
  iota_kernel<<<static_cast<unsigned>((c->n + 255) / 256), 256, 0, c->stream>>>(c->iota.as<int32_t>(), c->n);
  FSIL_LAUNCHED(c);
  int bits = 1;
  while ((int64_t(1) << bits) < c->k) ++bits;
  size_t tmp_bytes = 0;
  FSIL_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, c->dense.as<int32_t>(),
                                            c->sort_keys.as<int32_t>(), c->iota.as<int32_t>(),
                                            c->sort_vals.as<int32_t>(), n32, 0, bits, c->stream));
  c->sort_tmp.ensure(tmp_bytes);
  FSIL_CUDA(cub::DeviceRadixSort::SortPairs(c->sort_tmp.p, tmp_bytes, c->dense.as<int32_t>(),
                                            c->sort_keys.as<int32_t>(), c->iota.as<int32_t>(),
                                            c->sort_vals.as<int32_t>(), n32, 0, bits, c->stream));
  c->launches += 4;
  c->seg_start.ensure((2 * static_cast<size_t>(c->k) + 2) * sizeof(int64_t));
  int64_t* seg_begin = c->seg_start.as<int64_t>();
  int64_t* seg_end = seg_begin + c->k + 1;
  FSIL_CUDA(cudaMemsetAsync(seg_begin, 0, (2 * static_cast<size_t>(c->k) + 2) * sizeof(int64_t), c->stream));
  segment_bounds_kernel<<<static_cast<unsigned>((c->n + 255) / 256), 256, 0, c->stream>>>(
      c->sort_keys.as<int32_t>(), c->n, seg_begin, seg_end);
  FSIL_LAUNCHED(c);
  c->piece_start.ensure((2 * static_cast<size_t>(c->k) + 4) * sizeof(int64_t));
  int64_t* ppc = c->piece_start.as<int64_t>();
  int64_t* piece_start = ppc + c->k + 2;
  pieces_per_cluster_kernel<<<(c->k + 1 + 255) / 256, 256, 0, c->stream>>>(seg_begin, seg_end, c->k, ppc);
  FSIL_LAUNCHED(c);
  size_t scan_bytes = 0;
  FSIL_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, ppc, piece_start, c->k + 1, c->stream));
  if (scan_bytes > c->sort_tmp.bytes) c->sort_tmp.ensure(scan_bytes);
  FSIL_CUDA(cub::DeviceScan::ExclusiveSum(c->sort_tmp.p, scan_bytes, ppc, piece_start, c->k + 1, c->stream));
  c->launches += 1;
  const int64_t max_pieces = c->n / kPieceRows + c->k + 1;
  const int S1 = cos ? c->d + 1 : c->d + 2;
  c->partials.ensure(static_cast<size_t>(max_pieces) * S1 * sizeof(double));
  const int cpl_t = cpl <= 1 ? 1 : cpl <= 2 ? 2 : cpl <= 4 ? 4 : cpl <= 8 ? 8 : cpl <= 16 ? 16 : 32;
  if (cos)
    launch_pieces<true>(c, vec, cpl_t, max_pieces, lpr, c->sort_vals.as<int32_t>(), seg_begin,
                        seg_end, piece_start, c->partials.as<double>(), checks);
  else
    launch_pieces<false>(c, vec, cpl_t, max_pieces, lpr, c->sort_vals.as<int32_t>(), seg_begin,
                         seg_end, piece_start, c->partials.as<double>(), checks);
  const int64_t nthreads = static_cast<int64_t>(c->k) * S1;
  fold_pieces_kernel<<<static_cast<unsigned>((nthreads + 255) / 256), 256, 0, c->stream>>>(
      c->partials.as<double>(), piece_start, c->k, c->d, cos, stats);
  FSIL_LAUNCHED(c);
}

void derive(fsil_context* c) {
  const bool cos = c->metric == FSIL_COSINE;
  const int64_t kpad = ((c->k + 31) / 32) * 32;
  c->mu32.ensure(kpad * c->dp * sizeof(float));
  c->p32.ensure(kpad * sizeof(float));
  c->nk.ensure(kpad * sizeof(double));
  c->bound.ensure(4 * sizeof(float));
  FSIL_CUDA(cudaMemsetAsync(c->mu32.p, 0, kpad * c->dp * sizeof(float), c->stream));
  FSIL_CUDA(cudaMemsetAsync(c->p32.p, 0, kpad * sizeof(float), c->stream));
  FSIL_CUDA(cudaMemsetAsync(c->bound.p, 0, 4 * sizeof(float), c->stream));
  derive_kernel<<<c->k, 128, 0, c->stream>>>(c->stats_buf.as<double>(), c->k, c->d,
                                             static_cast<int>(c->dp), cos, c->mu32.as<float>(),
                                             c->p32.as<float>(), c->nk.as<double>(),
                                             c->bound.as<float>());
  FSIL_LAUNCHED(c);
}

}  // namespace fsil
