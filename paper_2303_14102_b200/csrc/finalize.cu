// finalize.cu -- K4 fp64 refinement of uncertified rows and K5 deterministic mean.
//
// K4 re-evaluates every foreign cluster of a flagged row in fp64 with the
// reference formulas and the reference's argmin rule (ascending k, strict <,
// so ties keep the lowest dense id: squared_euclidean.cpp:94-103,
// cosine.cpp:103-112), then rewrites a_i, b_i, s_i and the neighbour.
// K5 sums s_i in a fixed order (tile partials written by the scoring kernel,
// tiles that held refined rows re-summed from s[]), replacing the reference's
// serial left-to-right sum (report.cpp:36-40); the result is bit-identical run
// to run, and within ~1e-16 relative of the serial sum.
#include <algorithm>
#include <cstdlib>

#include "score_common.cuh"

namespace fsil {
namespace {

// One warp per flagged row.  x is staged once in shared memory (fp64); the warp walks
// the clusters 32 at a time: every lane accumulates partial dots over its dimensions
// (l = lane + 32 i, coalesced reads of each Y_k) for all 32 clusters, then a butterfly
// transpose-reduce leaves lane j holding the full dot of cluster kc + j (31 shuffles
// per 32 clusters instead of 5 per cluster).  Each lane keeps its ascending-k running
// argmin (strict <); the warp merge breaks ties towards the lowest k.
template <bool COS>
__device__ __forceinline__ void refine_rows(const ScoreParams& p, double* xs, int64_t warp, int64_t nwarps,
                                            int lane, const double* staged = nullptr) {
  const unsigned long long count = *p.flag_count;
  // cluster sums: staged in shared memory by the caller (small tables), else global
  const double* sums = staged ? staged : p.stats + (COS ? p.k : 2 * p.k);
  const int d = p.d, K = p.k;
  for (int64_t i = warp; i < static_cast<int64_t>(count); i += nwarps) {
    const int64_t row = p.flag_rows[i];
    const int64_t xo = row * d;
    const int own = p.dense[row];
    double ss = 0.0;
    __syncwarp();
    for (int l = lane; l < d; l += 32) {
      const double v = xval(p, xo + l);
      xs[l] = v;
      ss = fma(v, v, ss);
    }
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    __syncwarp();
    const double nrm = sqrt(ss);
    double best = INFINITY;
    int arg = -1;
    for (int kc = 0; kc < K; kc += 32) {
      double acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0;
      for (int l = lane; l < d; l += 32) {
        const double xv = xs[l];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int k = kc + j < K ? kc + j : K - 1;  // clamped; result unused
          acc[j] = fma(staged ? sums[static_cast<int64_t>(k) * d + l] : __ldg(sums + static_cast<int64_t>(k) * d + l), xv,
                       acc[j]);
        }
      }
#pragma unroll
      for (int sft = 16; sft >= 1; sft >>= 1) {  // transpose-reduce: acc[0] of lane j = cluster kc+j
        const bool up = (lane & sft) != 0;
#pragma unroll
        for (int j = 0; j < sft; ++j) {
          const double send = up ? acc[j] : acc[j + sft];
          const double keep = up ? acc[j + sft] : acc[j];
          acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
        }
      }
      const int k = kc + lane;
      if (k < K && k != own) {
        const double m = COS ? cos_foreign(p.nk[k], acc[0] / nrm) : sq_foreign(ss, p.stats[p.k + k], p.nk[k], acc[0]);
        if (m < best) {
          best = m;
          arg = k;
        }
      }
    }
    // warp argmin with ties broken towards the lowest k
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, off);
      if (oa >= 0 && (arg < 0 || ob < best || (ob == best && oa < arg))) {
        best = ob;
        arg = oa;
      }
    }
    // own-cluster mean, dims split over lanes
    const double* yo = sums + static_cast<int64_t>(own) * d;
    double co = 0.0;
    for (int l = lane; l < d; l += 32) co = fma(yo[l], xs[l], co);
    for (int off = 16; off > 0; off >>= 1) co += __shfl_xor_sync(0xffffffffu, co, off);
    if (lane == 0) {
      const double n_o = p.nk[own];
      const bool singleton = n_o == 1.0;
      double a = 0.0;
      if (!singleton) a = COS ? cos_own(n_o, co / nrm) : sq_own(ss, p.stats[p.k + own], n_o, co);
      const double s = singleton ? 0.0 : assemble_score(a, best);
      p.s[row] = s;
      if (p.nb) p.nb[row] = arg;
      if (p.own) p.own[row] = own;
      if (p.a) p.a[row] = a;
      if (p.b) p.b[row] = best;
    }
  }
}

template <bool COS>
__global__ void __launch_bounds__(256) refine_kernel(ScoreParams p) {
  if (*p.abort) return;
  extern __shared__ double xs_all[];  // [warps per block][d]
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  refine_rows<COS>(p, xs_all + static_cast<int64_t>(threadIdx.x >> 5) * p.d, warp, nwarps, threadIdx.x & 31);
}

// Tiled fp64 refinement for many flagged rows against many clusters (C4, C5): a block
// takes 32 flagged rows and walks the clusters 64 at a time, D in chunks of 32, with
// the row and cluster-mean tiles staged in shared memory (each mean tile is read once
// per 32 rows instead of once per row).  Thread (ty, tx) owns rows 2ty, 2ty+1 and
// clusters tx + 16 j of each tile: ascending per thread, strict < -- then the 16
// threads of a row merge with ties to the lowest k (the reference's rule).
//
// Few flagged rows (C5: ~1e2 of 1e7) would leave most of the grid idle, one block walking
// all K clusters per 32 rows: the cluster range is then split into nsl slices (units =
// row tiles x slices, nsl chosen on the device from the flagged count so the units cover
// the grid).  A unit writes its rows' slice minimum (ties already at the lowest k); the
// last unit of a row tile to finish (ticket) merges the slices in ascending order -- strict
// <, so the lowest k keeps ties across slices too -- and finalises the rows.
constexpr int kRT = 32, kCT = 64, kDC = 32;
struct RefineSplit {
  double* best;   // [row tiles * 32][nsl] slice minima (nsl > 1 only: < 2 * grid * 32 entries)
  int* arg;
  unsigned* cnt;  // [grid] per-row-tile tickets, zero between launches (the merger resets)
};
template <bool COS>
__global__ void __launch_bounds__(256) refine_tiled_kernel(ScoreParams p, RefineSplit rs) {
  if (*p.abort) return;
  __shared__ double xs[kRT][kDC + 1];
  __shared__ double ys[kCT][kDC + 1];
  __shared__ double s_ss[kRT], s_co[kRT], s_best[kRT][17];
  __shared__ int s_arg[kRT][17], s_own[kRT];
  __shared__ int64_t s_row[kRT];
  __shared__ bool s_last;
  const int64_t count = static_cast<int64_t>(*p.flag_count);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4, lane = tid & 31, warp = tid >> 5;
  const double* sums = p.stats + (COS ? p.k : 2 * p.k);
  const int d = p.d, K = p.k;
  const int64_t rtiles = (count + kRT - 1) / kRT;
  const int nct = (K + kCT - 1) / kCT;
  const int nsl = rtiles >= static_cast<int64_t>(gridDim.x) ? 1 : static_cast<int>(min(static_cast<int64_t>(nct), (static_cast<int64_t>(gridDim.x) + rtiles - 1) / rtiles));
  const int64_t nunits = rtiles * nsl;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t tile = u / nsl;
    const int sl = static_cast<int>(u % nsl);
    const int64_t t0 = tile * kRT;
    const int c_lo = (sl * nct / nsl) * kCT, c_hi = min(K, ((sl + 1) * nct / nsl) * kCT);
    __syncthreads();
    if (tid < kRT) {
      const int64_t i = t0 + tid;
      const int64_t row = i < count ? p.flag_rows[i] : -1;
      s_row[tid] = row;
      s_own[tid] = row >= 0 ? p.dense[row] : -1;
      s_co[tid] = 0.0;
    }
    __syncthreads();
    for (int r = warp; r < kRT; r += 8) {  // ||x||^2 and the own-cluster dot per row
      const int64_t row = s_row[r];
      double ss = 0.0, co = 0.0;
      if (row >= 0) {
        const int64_t xo = row * d;
        const double* yo = sums + static_cast<int64_t>(s_own[r]) * d;
        for (int l = lane; l < d; l += 32) {
          const double v = xval(p, xo + l);
          ss = fma(v, v, ss);
          co = fma(yo[l], v, co);
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, off);
        co += __shfl_xor_sync(0xffffffffu, co, off);
      }
      if (lane == 0) {
        s_ss[r] = ss;
        s_co[r] = co;
      }
    }
    __syncthreads();
    const int r0 = 2 * ty, r1 = 2 * ty + 1;
    const double ss0 = s_ss[r0], ss1 = s_ss[r1];
    const double nrm0 = sqrt(ss0), nrm1 = sqrt(ss1);
    const int own0 = s_own[r0], own1 = s_own[r1];
    double best0 = INFINITY, best1 = INFINITY;
    int arg0 = -1, arg1 = -1;
    for (int c0 = c_lo; c0 < c_hi; c0 += kCT) {
      double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
      for (int l0 = 0; l0 < d; l0 += kDC) {
        __syncthreads();
        for (int e = tid; e < kRT * kDC; e += 256) {  // rows (fp32 -> fp64), zero padded
          const int r = e / kDC, l = e % kDC;
          const int64_t row = s_row[r];
          xs[r][l] = (row >= 0 && l0 + l < d) ? xval(p, row * d + l0 + l) : 0.0;
        }
        for (int e = tid; e < kCT * kDC; e += 256) {  // cluster sums, coalesced along D
          const int c = e / kDC, l = e % kDC;
          ys[c][l] = (c0 + c < K && l0 + l < d) ? sums[static_cast<int64_t>(c0 + c) * d + l0 + l] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int l = 0; l < kDC; ++l) {
          const double xa = xs[r0][l], xb = xs[r1][l];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double y = ys[tx + 16 * j][l];
            acc[0][j] = fma(y, xa, acc[0][j]);
            acc[1][j] = fma(y, xb, acc[1][j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k = c0 + tx + 16 * j;
        if (k >= K) continue;
        const double nk = p.nk[k];
        if (k != own0) {
          const double m = COS ? cos_foreign(nk, acc[0][j] / nrm0) : sq_foreign(ss0, p.stats[K + k], nk, acc[0][j]);
          if (m < best0) {
            best0 = m;
            arg0 = k;
          }
        }
        if (k != own1) {
          const double m = COS ? cos_foreign(nk, acc[1][j] / nrm1) : sq_foreign(ss1, p.stats[K + k], nk, acc[1][j]);
          if (m < best1) {
            best1 = m;
            arg1 = k;
          }
        }
      }
    }
    s_best[r0][tx] = best0;
    s_arg[r0][tx] = arg0;
    s_best[r1][tx] = best1;
    s_arg[r1][tx] = arg1;
    __syncthreads();
    double best = INFINITY;
    int arg = -1;
    if (tid < kRT) {
      for (int j = 0; j < 16; ++j) {  // lowest k among equal minima
        const double b = s_best[tid][j];
        const int a = s_arg[tid][j];
        if (a >= 0 && (arg < 0 || b < best || (b == best && a < arg))) {
          best = b;
          arg = a;
        }
      }
    }
    if (nsl > 1) {
      if (tid < kRT) {
        rs.best[(t0 + tid) * nsl + sl] = best;
        rs.arg[(t0 + tid) * nsl + sl] = arg;
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) s_last = atomicAdd(rs.cnt + tile, 1u) == static_cast<unsigned>(nsl - 1);
      __syncthreads();
      if (!s_last) continue;
      __threadfence();
      if (tid == 0) rs.cnt[tile] = 0u;  // ready for the next launch
      if (tid < kRT) {
        best = INFINITY;
        arg = -1;
        for (int q = 0; q < nsl; ++q) {  // ascending slices: strict < keeps the lowest k
          const double b = __ldcg(rs.best + (t0 + tid) * nsl + q);
          const int a = __ldcg(rs.arg + (t0 + tid) * nsl + q);
          if (a >= 0 && (arg < 0 || b < best)) {
            best = b;
            arg = a;
          }
        }
      }
    }
    if (tid < kRT) {
      const int r = tid;
      const int64_t row = s_row[r];
      if (row >= 0) {
        const int own = s_own[r];
        const double n_o = p.nk[own];
        const bool singleton = n_o == 1.0;
        double a = 0.0;
        if (!singleton)
          a = COS ? cos_own(n_o, s_co[r] / sqrt(s_ss[r])) : sq_own(s_ss[r], p.stats[K + own], n_o, s_co[r]);
        p.s[row] = singleton ? 0.0 : assemble_score(a, best);
        if (p.nb) p.nb[row] = arg;
        if (p.own) p.own[row] = own;
        if (p.a) p.a[row] = a;
        if (p.b) p.b[row] = best;
      }
    }
  }
}

// Group partials: a block covers 32 tiles (one warp per 4 tiles); tiles that held
// refined rows are re-summed from s[] by the warp (fixed lane order + xor tree);
// then a fixed-order tree over the 32 tile values.  The last block to finish (atomic
// ticket) sums the group partials in a fixed order into result[] and, on a single
// GPU, writes the call's summary straight into mapped host memory.
struct TotalArgs {
  double* group_sum;
  double* result;                        // [0] sum s_i, [1] flagged rows, [2] exact rows
  const unsigned long long* flag_count;
  const unsigned long long* exact_count;  // null if unused
  const unsigned long long* pair_count;   // tcgen05 top-3 certified pairs (null if unused)
  unsigned int* ticket;                   // zero on entry; reset by the last block
  HostSummary* hsum;                      // single GPU: summary target (null in shard mode)
  const int64_t* checks;
  const int* missing;
};

// One group of kGroupTiles (64) tiles by a 256-thread block -- C2's 7,813 tiles make 123
// groups, one round over 148 blocks; true in the block that completed the last of
// `ngroups` groups (it then sums them: tile_total).
constexpr int kGroupTiles = 64;
__device__ __forceinline__ bool tile_group_one(const double* __restrict__ tile_sum,
                                               const int32_t* __restrict__ tile_flag, const double* s,
                                               int64_t ntiles, int tile_rows, int64_t n, const TotalArgs& ta,
                                               int64_t g, int64_t ngroups) {
  __shared__ double sm[kGroupTiles];
  __shared__ int fl[kGroupTiles];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = g * kGroupTiles;
  if (threadIdx.x < kGroupTiles) {  // every tile's flag and partial in one round trip
    const int64_t tt = t0 + threadIdx.x;
    const bool in = tt < ntiles;
    fl[threadIdx.x] = in ? tile_flag[tt] : 0;
    sm[threadIdx.x] = in ? tile_sum[tt] : 0.0;
  }
  __syncthreads();
  for (int j = warp; j < kGroupTiles; j += 8) {  // tiles that held refined rows: re-sum from s[]
    if (!fl[j]) continue;
    const int64_t tt = t0 + j;
    const int64_t r0 = tt * tile_rows, r1 = min(n, r0 + tile_rows);
    double acc = 0.0;
    for (int64_t r = r0 + lane; r < r1; r += 32) acc += __ldcg(s + r);  // written by this grid
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) sm[j] = acc;
  }
  __syncthreads();
  if (warp == 0) {
    double v = sm[lane] + sm[lane + 32];  // fixed pairing, then a fixed xor tree
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) {
      ta.group_sum[g] = v;
      __threadfence();
      last = atomicAdd(ta.ticket, 1u) == static_cast<unsigned>(ngroups - 1);
    }
  }
  __syncthreads();
  const bool l = last;
  __syncthreads();  // `last` is rewritten by the block's next group
  return l;
}

__device__ __forceinline__ void tile_total(const TotalArgs& ta, int64_t ngroups) {
  __shared__ double red[256];
  __threadfence();
  // fixed order: thread i sums groups i, i + 256, ...; then a fixed tree
  double acc = 0.0;
  for (int64_t g = threadIdx.x; g < ngroups; g += 256) acc += __ldcg(ta.group_sum + g);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int stride = 128; stride > 0; stride >>= 1) {
    if (threadIdx.x < stride) red[threadIdx.x] += red[threadIdx.x + stride];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double flagged = static_cast<double>(*ta.flag_count);
    const double exact = ta.exact_count ? static_cast<double>(*ta.exact_count) : 0.0;
    ta.result[0] = red[0];
    ta.result[1] = flagged;
    ta.result[2] = exact;
    if (ta.hsum) {
      ta.hsum->checks[0] = ta.checks[0];
      ta.hsum->checks[1] = ta.checks[1];
      ta.hsum->missing = *ta.missing;
      ta.hsum->result[0] = red[0];
      ta.hsum->result[1] = flagged;
      ta.hsum->result[2] = exact;
    }
    *ta.ticket = 0u;
  }
}

__global__ void __launch_bounds__(256) tile_group_kernel(const double* __restrict__ tile_sum,
                                                         const int32_t* __restrict__ tile_flag,
                                                         const double* __restrict__ s,
                                                         int64_t ntiles, int tile_rows, int64_t n,
                                                         TotalArgs ta) {
  if (tile_group_one(tile_sum, tile_flag, s, ntiles, tile_rows, n, ta, blockIdx.x, gridDim.x))
    tile_total(ta, gridDim.x);
}

// FSIL_PATH_FP64: every row goes through the fp64 re-evaluation.
__global__ void flag_all_kernel(int64_t n, int tile_rows, int32_t* flag_rows, int32_t* tile_flag,
                                double* tile_sum, unsigned long long* flag_count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) flag_rows[i] = static_cast<int32_t>(i);
  if (i < (n + tile_rows - 1) / tile_rows) {
    tile_flag[i] = 1;
    tile_sum[i] = 0.0;
  }
  if (i == 0) *flag_count = static_cast<unsigned long long>(n);
}

// The whole post-scoring phase of the FFMA and fp64 paths in one cooperative launch
// (small cluster tables): flagged rows, grid barrier, then the tile groups and -- in the
// block that finishes the last group -- the fixed-order total.
template <bool COS>
__global__ void __launch_bounds__(256) post_kernel(ScoreParams p, int64_t ntiles, int tile_rows, TotalArgs ta,
                                                   unsigned int* bar, bool stage) {
  griddep_wait();  // (PDL) the scoring kernel's rows, flags and tile sums are visible
  extern __shared__ double xs_all[];  // [8 warps][d], then (stage) the cluster sums [K][d]
  const bool abort = *p.abort != 0;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  double* staged = nullptr;
  // blocks whose warps have no flagged row skip the table (a handful of flagged rows:
  // a handful of blocks do any per-row work)
  if (stage) {
    const int64_t w0 = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5);
    stage = w0 < static_cast<int64_t>(*p.flag_count);
  }
  if (stage) {  // the table in shared memory: its loads overlap the first rows' own
    staged = xs_all + 8 * p.d;
    const double* sums = p.stats + (COS ? p.k : 2 * p.k);
    for (int64_t e = threadIdx.x; e < static_cast<int64_t>(p.k) * p.d; e += blockDim.x) staged[e] = __ldg(sums + e);
    __syncthreads();
  }
  if (!abort) refine_rows<COS>(p, xs_all + static_cast<int64_t>(threadIdx.x >> 5) * p.d, warp, nwarps, lane, staged);
  grid_barrier(bar, bar + 1);
  const int64_t ngroups = (ntiles + kGroupTiles - 1) / kGroupTiles > 0 ? (ntiles + kGroupTiles - 1) / kGroupTiles : 1;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x)
    if (tile_group_one(p.tile_sum, p.tile_flag, p.s, ntiles, tile_rows, p.n, ta, g, ngroups)) tile_total(ta, ngroups);
}

// ---------------------------------------------------------------- exact pass ----
// Every row's a_i, b_i and s_i in fp64 from its own cluster and its (certified or
// refined) neighbour: three length-D dots -- ||x||^2, Y_own.x, Y_nb.x -- and the
// reference formulas (squared_euclidean.cpp:77-81, cosine.cpp:83-87, report.cpp:7-30).
// The tensor-core pass only nominates the neighbour, so nothing that reaches s_i or S
// carries tensor-core rounding: the fp32 input widened exactly, fp64 products and sums.
//
// LPR lanes per row, each owning CPL element pairs (D = 2 LPR CPL; CPL = 0: any even D):
// x read as pairs (coalesced along the row), the cluster sums as double2 from shared
// memory (the table staged once per CTA when it fits) or from L2.  Work unit: 32
// consecutive rows per warp, two row passes' loads in flight; the unit's s_i are summed
// in a fixed order into usum[u], and the CTA that finishes last (atomic ticket) sums the
// units in a fixed order, so S is bit-identical run to run.
constexpr int kUnitRows = 32;
constexpr int kExactThreads = 512;

template <typename T>
struct PairOf;
template <>
struct PairOf<float> {
  using V = float2;
};
template <>
struct PairOf<double> {
  using V = double2;
};

struct ExactArgs {
  double* usum;       // [nunits] fixed-order sums of s_i over 32-row units
  int64_t nunits;
  TotalArgs ta;
  unsigned int* bar;  // grid-barrier words (cooperative launch with the refinement phase)
  const int2* pairs;  // certified pairs (resolved with the refinement phase)
  int refine;         // 1: refine the flagged rows first (cooperative launch), then barrier
  int stage;          // 1: the cluster-sum table is staged in shared memory
  const int32_t* order;  // rows in label-sorted order (sorted aggregation path), or null:
                         // consecutive positions then share their own cluster's sums (cache
                         // reuse of the fp64 table rows); units are runs of positions
};

template <bool COS>
__device__ __forceinline__ double exact_finish(const ScoreParams& p, int64_t row, int own, int nb, double ss,
                                               double co, double cb) {
  const double n_o = p.nk[own], n_b = p.nk[nb];
  const bool singleton = n_o == 1.0;
  double a, b;
  if (COS) {
    const double nrm = sqrt(ss);
    b = cos_foreign(n_b, cb / nrm);
    a = singleton ? 0.0 : cos_own(n_o, co / nrm);
  } else {
    b = sq_foreign(ss, p.stats[p.k + nb], n_b, cb);
    a = singleton ? 0.0 : sq_own(ss, p.stats[p.k + own], n_o, co);
  }
  const double s = singleton ? 0.0 : assemble_score(a, b);
  p.s[row] = s;
  if (p.a) p.a[row] = a;
  if (p.b) p.b[row] = b;
  if (p.own) p.own[row] = own;
  return s;
}

template <bool COS, typename T, int LPR, int CPL>
__device__ __forceinline__ void exact_units(const ScoreParams& p, const double* ytab, double* __restrict__ usum,
                                            int64_t nunits, int64_t wid, int64_t nw, int lane,
                                            const int32_t* __restrict__ order) {
  using V = typename PairOf<T>::V;
  constexpr int RPP = 32 / LPR;           // rows per pass
  constexpr int PPU = kUnitRows / RPP;    // passes per unit (= LPR)
  const int sub = lane / LPR, li = lane % LPR;
  const int d = p.d, d2 = p.d >> 1;
  const T* X = sizeof(T) == 8 ? reinterpret_cast<const T*>(p.X64) : reinterpret_cast<const T*>(p.X);
  if (wid >= nunits) return;
  if constexpr (CPL > 0 && CPL <= 4 && LPR <= 8) {
    // Narrow rows (D <= 64: LPR <= 8 lanes per row and passes per unit, at most four pairs per
    // lane; measured at D = 128 the 48 live partials spill and the plain ring below wins).  Same rolling register ring
    // as below, but the LPR lanes' partial dots of every pass are kept until the unit ends and
    // reduced by a transposing butterfly: at each step a lane hands half of its passes to its
    // partner and keeps the other half, so after log2(LPR) steps lane (sub, li) holds the full
    // sums of pass li's row -- (LPR - 1) 64-bit exchanges per quantity and unit instead of
    // PPU log2(LPR) + PPU (the pass was shuffle- and issue-bound at D <= 128, not HBM-bound).
    // The pairing (li ^ LPR/2, ..., li ^ 1) is the plain butterfly's, so each row's sums are
    // bit-identical to it.
    constexpr int DEPTH = 4;
    static_assert(PPU % DEPTH == 0 && PPU == LPR, "a unit must end on a ring boundary");
    const int64_t npass = ((nunits - 1 - wid) / nw + 1) * PPU;
    V buf[DEPTH][CPL];
    int bown[DEPTH], bnb[DEPTH];
    auto row_of = [&](int64_t j) { return (wid + (j / PPU) * nw) * kUnitRows + (j % PPU) * RPP + sub; };
    auto load = [&](int64_t j, V (&b)[CPL], int& o, int& nb) {
      const int64_t pos = row_of(j);
      const bool ok = j < npass && pos < p.n;
      const V* xr = reinterpret_cast<const V*>(X + (ok ? pos : 0) * d);
#pragma unroll
      for (int c = 0; c < CPL; ++c) b[c] = xr[li + LPR * c];
      o = ok ? __ldg(p.dense + pos) : 0;
      nb = ok ? p.nb[pos] : 0;
    };
#pragma unroll
    for (int h = 0; h < DEPTH; ++h) load(h, buf[h], bown[h], bnb[h]);
    for (int64_t j0 = 0; j0 < npass; j0 += PPU) {
      double pss[PPU], pco[PPU], pcb[PPU];
      int rown = 0, rnb = 0;
#pragma unroll
      for (int ps = 0; ps < PPU; ++ps) {
        constexpr int kD = DEPTH;
        const int h = ps % kD;
        const int own = bown[h], nb = bnb[h];
        const double* yo = ytab + static_cast<int64_t>(own) * d;
        const double* yb = ytab + static_cast<int64_t>(nb) * d;
        double ss = 0.0, co = 0.0, cb = 0.0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int q = li + LPR * c;
          const double2 o = *reinterpret_cast<const double2*>(yo + 2 * q);
          const double2 b = *reinterpret_cast<const double2*>(yb + 2 * q);
          const double x0 = static_cast<double>(buf[h][c].x), x1 = static_cast<double>(buf[h][c].y);
          ss = fma(x0, x0, ss);
          ss = fma(x1, x1, ss);
          co = fma(o.x, x0, co);
          co = fma(o.y, x1, co);
          cb = fma(b.x, x0, cb);
          cb = fma(b.y, x1, cb);
        }
        pss[ps] = ss;
        pco[ps] = co;
        pcb[ps] = cb;
        if (li == ps) {  // (every lane of the row's group loaded its own / neighbour ids)
          rown = own;
          rnb = nb;
        }
        load(j0 + ps + DEPTH, buf[h], bown[h], bnb[h]);  // refill the slot just consumed
      }
      // transposing butterfly: `half` passes survive each step; the lane keeps the passes whose
      // bit matches its own li bit
#pragma unroll
      for (int half = LPR >> 1; half > 0; half >>= 1) {
        const bool up = (li & half) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
          const double s0 = up ? pss[i] : pss[i + half], s1 = up ? pco[i] : pco[i + half],
                       s2 = up ? pcb[i] : pcb[i + half];
          const double k0 = up ? pss[i + half] : pss[i], k1 = up ? pco[i + half] : pco[i],
                       k2 = up ? pcb[i + half] : pcb[i];
          pss[i] = k0 + __shfl_xor_sync(0xffffffffu, s0, half);
          pco[i] = k1 + __shfl_xor_sync(0xffffffffu, s1, half);
          pcb[i] = k2 + __shfl_xor_sync(0xffffffffu, s2, half);
        }
      }
      // lane (sub, li) holds row li * RPP + sub of the unit; fixed-order tree over the lanes
      const int64_t u = wid + (j0 / PPU) * nw;
      const int64_t pos = u * kUnitRows + li * RPP + sub;
      double su = pos < p.n ? exact_finish<COS>(p, pos, rown, rnb, pss[0], pco[0], pcb[0]) : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) su += __shfl_xor_sync(0xffffffffu, su, off);
      if (lane == 0) usum[u] = su;
    }
  } else if constexpr (CPL > 0) {
    // The warp's passes (units wid, wid + nw, ...; PPU passes each) form one stream with a
    // rolling register ring: pass j + DEPTH is loaded while pass j is reduced, so DEPTH
    // passes' rows are always in flight (the pass is HBM-latency bound otherwise).
    constexpr int DEPTH = CPL >= 8 ? 2 : 4;
    static_assert(PPU % DEPTH == 0, "a unit must end on a ring boundary");
    const int64_t npass = ((nunits - 1 - wid) / nw + 1) * PPU;
    V buf[DEPTH][CPL];
    int bown[DEPTH], bnb[DEPTH];
    // after the unit's PPU passes, lane L holds row L's three dots: the fp64 finish (five
    // divisions) then runs once per unit with every lane active, and s_i is stored coalesced
    double rss = 0.0, rco = 0.0, rcb = 0.0;
    int rown = 0, rnb = 0;
    const int src_lane = (lane % RPP) * LPR;  // group leader holding row (pass * RPP + lane % RPP)
    auto row_of = [&](int64_t j) { return (wid + (j / PPU) * nw) * kUnitRows + (j % PPU) * RPP + sub; };
    auto load = [&](int64_t j, V (&b)[CPL], int& o, int& nb) {
      const int64_t pos = row_of(j);
      const bool ok = j < npass && pos < p.n;
      const int64_t row = ok && order ? static_cast<int64_t>(__ldg(order + pos)) : pos;
      const V* xr = reinterpret_cast<const V*>(X + (ok ? row : 0) * d);
#pragma unroll
      for (int c = 0; c < CPL; ++c) b[c] = xr[li + LPR * c];
      o = ok ? __ldg(p.dense + row) : 0;
      nb = ok ? p.nb[row] : 0;
    };
#pragma unroll
    for (int h = 0; h < DEPTH; ++h) load(h, buf[h], bown[h], bnb[h]);
    for (int64_t j0 = 0; j0 < npass; j0 += DEPTH) {
#pragma unroll
      for (int h = 0; h < DEPTH; ++h) {
        const int64_t j = j0 + h;
        const int own = bown[h], nb = bnb[h];
        const double* yo = ytab + static_cast<int64_t>(own) * d;
        const double* yb = ytab + static_cast<int64_t>(nb) * d;
        double ss = 0.0, co = 0.0, cb = 0.0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int q = li + LPR * c;
          const double2 o = *reinterpret_cast<const double2*>(yo + 2 * q);
          const double2 b = *reinterpret_cast<const double2*>(yb + 2 * q);
          const double x0 = static_cast<double>(buf[h][c].x), x1 = static_cast<double>(buf[h][c].y);
          ss = fma(x0, x0, ss);
          ss = fma(x1, x1, ss);
          co = fma(o.x, x0, co);
          co = fma(o.y, x1, co);
          cb = fma(b.x, x0, cb);
          cb = fma(b.y, x1, cb);
        }
        load(j + DEPTH, buf[h], bown[h], bnb[h]);  // refill the slot just consumed
#pragma unroll
        for (int off = LPR >> 1; off > 0; off >>= 1) {
          ss += __shfl_xor_sync(0xffffffffu, ss, off);
          co += __shfl_xor_sync(0xffffffffu, co, off);
          cb += __shfl_xor_sync(0xffffffffu, cb, off);
        }
        const double vss = __shfl_sync(0xffffffffu, ss, src_lane), vco = __shfl_sync(0xffffffffu, co, src_lane),
                     vcb = __shfl_sync(0xffffffffu, cb, src_lane);
        const int vown = __shfl_sync(0xffffffffu, own, src_lane), vnb = __shfl_sync(0xffffffffu, nb, src_lane);
        if (lane / RPP == static_cast<int>(j % PPU)) {
          rss = vss;
          rco = vco;
          rcb = vcb;
          rown = vown;
          rnb = vnb;
        }
      }
      if ((j0 + DEPTH) % PPU == 0) {  // a unit ends here: one row per lane, fixed-order tree
        const int64_t u = wid + ((j0 + DEPTH) / PPU - 1) * nw;
        const int64_t pos = u * kUnitRows + lane;
        const int64_t row = pos < p.n && order ? static_cast<int64_t>(__ldg(order + pos)) : pos;
        double su = pos < p.n ? exact_finish<COS>(p, row, rown, rnb, rss, rco, rcb) : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) su += __shfl_xor_sync(0xffffffffu, su, off);
        if (lane == 0) usum[u] = su;
      }
    }
  } else {  // any even D: one row per pass, LPR lanes stride the pairs
    for (int64_t u = wid; u < nunits; u += nw) {
      const int64_t r0 = u * kUnitRows;
      double su = 0.0;
#pragma unroll 1
      for (int pass = 0; pass < PPU; ++pass) {
        const int64_t pos = r0 + pass * RPP + sub;
        const bool ok = pos < p.n;
        const int64_t row = ok && order ? static_cast<int64_t>(__ldg(order + pos)) : pos;
        const V* xr = reinterpret_cast<const V*>(X + (ok ? row : 0) * d);
        const int own = ok ? __ldg(p.dense + row) : 0, nb = ok ? p.nb[row] : 0;
        const double* yo = ytab + static_cast<int64_t>(own) * d;
        const double* yb = ytab + static_cast<int64_t>(nb) * d;
        double ss = 0.0, co = 0.0, cb = 0.0;
        for (int q = li; q < d2; q += LPR) {
          const V xv = xr[q];
          const double x0 = static_cast<double>(xv.x), x1 = static_cast<double>(xv.y);
          ss = fma(x0, x0, ss);
          ss = fma(x1, x1, ss);
          co = fma(yo[2 * q], x0, co);
          co = fma(yo[2 * q + 1], x1, co);
          cb = fma(yb[2 * q], x0, cb);
          cb = fma(yb[2 * q + 1], x1, cb);
        }
#pragma unroll
        for (int off = LPR >> 1; off > 0; off >>= 1) {
          ss += __shfl_xor_sync(0xffffffffu, ss, off);
          co += __shfl_xor_sync(0xffffffffu, co, off);
          cb += __shfl_xor_sync(0xffffffffu, cb, off);
        }
        if (li == 0 && ok) su += exact_finish<COS>(p, row, own, nb, ss, co, cb);
      }
#pragma unroll
      for (int off = 16; off >= LPR; off >>= 1) su += __shfl_xor_sync(0xffffffffu, su, off);
      if (lane == 0) usum[u] = su;
    }
  }
}

// Fixed-order total of the unit sums by the last CTA (kExactThreads threads).
__device__ __forceinline__ void unit_total(const ExactArgs& ea, int64_t exact_rows) {
  __shared__ double red[kExactThreads];
  __threadfence();
  double acc = 0.0;
  for (int64_t u = threadIdx.x; u < ea.nunits; u += kExactThreads) acc += __ldcg(ea.usum + u);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int stride = kExactThreads / 2; stride > 0; stride >>= 1) {
    if (threadIdx.x < stride) red[threadIdx.x] += red[threadIdx.x + stride];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const TotalArgs& ta = ea.ta;
    const double flagged = static_cast<double>(*ta.flag_count);
    const double exact = static_cast<double>(exact_rows);
    // (certified pairs + the threshold mode's three/four-candidate records)
    const double pairs = ta.pair_count ? static_cast<double>(ta.pair_count[0] + ta.pair_count[1]) : 0.0;
    ta.result[0] = red[0];
    ta.result[1] = flagged;
    ta.result[2] = exact;
    ta.result[3] = pairs;
    if (ta.hsum) {
      ta.hsum->checks[0] = ta.checks[0];
      ta.hsum->checks[1] = ta.checks[1];
      ta.hsum->missing = *ta.missing;
      ta.hsum->result[0] = red[0];
      ta.hsum->result[1] = flagged;
      ta.hsum->result[2] = exact;
      ta.hsum->result[3] = pairs;
    }
    *ta.ticket = 0u;
  }
}

// Certified pairs (tcgen05 top-3): the neighbour is one of two columns {nb[row], c2}.
// One warp per pair: the two fp64 foreign means with the reference formula, clamp
// included, then the reference's rule -- strict <, equal means keep the lower index
// (squared_euclidean.cpp:94-103, cosine.cpp:103-112).
template <bool COS>
__device__ __forceinline__ void pair_rows_body(const ScoreParams& p, const int2* __restrict__ pairs,
                                               const unsigned long long* count, const double* sums, int64_t warp,
                                               int64_t nwarps, int lane) {
  const int64_t cnt = static_cast<int64_t>(*count);
  const int d = p.d;
  // fp32 rows and fp64 sums in 16-byte units: D a multiple of 4 and both bases aligned
  const bool vec = p.X64 == nullptr && (d & 3) == 0 && ((reinterpret_cast<uintptr_t>(p.X) | reinterpret_cast<uintptr_t>(sums)) & 15) == 0;
  for (int64_t i = warp; i < cnt; i += nwarps) {
    const int2 pr = pairs[i];
    const int64_t row = pr.x;
    const int c1 = p.nb[row], c2 = pr.y;
    const double* y1 = sums + static_cast<int64_t>(c1) * d;
    const double* y2 = sums + static_cast<int64_t>(c2) * d;
    double ss = 0.0, d1 = 0.0, d2 = 0.0;
    if (vec) {  // 16-byte loads, four elements per lane and step (wide rows: the loads in flight
                // set this pass's time, 15 KB per pair from L2)
      const float* xr = p.X + row * d;
#pragma unroll 2
      for (int l = lane * 4; l < d; l += 128) {
        const float4 xv = *reinterpret_cast<const float4*>(xr + l);
        const double2 a0 = *reinterpret_cast<const double2*>(y1 + l), a1 = *reinterpret_cast<const double2*>(y1 + l + 2);
        const double2 b0 = *reinterpret_cast<const double2*>(y2 + l), b1 = *reinterpret_cast<const double2*>(y2 + l + 2);
        const double x0 = xv.x, x1 = xv.y, x2 = xv.z, x3 = xv.w;
        ss = fma(x0, x0, ss);
        ss = fma(x1, x1, ss);
        ss = fma(x2, x2, ss);
        ss = fma(x3, x3, ss);
        d1 = fma(a0.x, x0, d1);
        d1 = fma(a0.y, x1, d1);
        d1 = fma(a1.x, x2, d1);
        d1 = fma(a1.y, x3, d1);
        d2 = fma(b0.x, x0, d2);
        d2 = fma(b0.y, x1, d2);
        d2 = fma(b1.x, x2, d2);
        d2 = fma(b1.y, x3, d2);
      }
    } else {
      for (int l = lane; l < d; l += 32) {
        const double v = xval(p, row * d + l);
        ss = fma(v, v, ss);
        d1 = fma(y1[l], v, d1);
        d2 = fma(y2[l], v, d2);
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      ss += __shfl_xor_sync(0xffffffffu, ss, off);
      d1 += __shfl_xor_sync(0xffffffffu, d1, off);
      d2 += __shfl_xor_sync(0xffffffffu, d2, off);
    }
    if (lane == 0) {
      double m1, m2;
      if (COS) {
        const double nrm = sqrt(ss);
        m1 = cos_foreign(p.nk[c1], d1 / nrm);
        m2 = cos_foreign(p.nk[c2], d2 / nrm);
      } else {
        m1 = sq_foreign(ss, p.stats[p.k + c1], p.nk[c1], d1);
        m2 = sq_foreign(ss, p.stats[p.k + c2], p.nk[c2], d2);
      }
      p.nb[row] = (m2 < m1 || (m2 == m1 && c2 < c1)) ? c2 : c1;
    }
  }
}

// Threshold mode's resolution pass.  The scoring epilogue left in the top bits of nb[row]:
// 0 the neighbour is certain; 2..4 the neighbour is one of that many columns -- nb[row] and
// cand[row].{x,y,z}; 1 no usable candidate set.  This pass scans nb (128 rows per warp step), and
// the warp resolves its marked rows four at a time (eight lanes each): the candidates' fp64 foreign means
// with the reference formula, clamp included, then the reference's rule -- strict <, equal
// means keep the lowest index (squared_euclidean.cpp:94-103) -- or, for code 1, the row
// joins the fp64 refinement's list.  counts[1] += rows resolved here (statistics).
template <bool COS>
__global__ void __launch_bounds__(256) thr_resolve_kernel(ScoreParams p, const int4* __restrict__ cand,
                                                          unsigned long long* counts) {
  griddep_wait();
  if (*p.abort) return;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31, sub = lane >> 3, li = lane & 7;
  const double* sums = p.stats + (COS ? p.k : 2 * p.k);
  const int d = p.d;
  const bool vec = p.X64 == nullptr && (d & 3) == 0 && ((reinterpret_cast<uintptr_t>(p.X) | reinterpret_cast<uintptr_t>(sums)) & 15) == 0;
  unsigned long long resolved = 0;
  // 128 consecutive rows per warp step (four nb loads in flight); their marked rows are
  // resolved four at a time, eight lanes each: the chain per row -- record, row and candidate
  // sums loads, reduction, fp64 finish -- is latency, so rows overlap
  for (int64_t base = warp * 128; base < p.n; base += nwarps * 128) {
    uint32_t v[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int64_t mine = base + g * 32 + lane;
      v[g] = mine < p.n ? static_cast<uint32_t>(p.nb[mine]) : 0u;
    }
    unsigned long long todo_lo = __ballot_sync(0xffffffffu, (v[0] >> 28) != 0u) |
                                 (static_cast<unsigned long long>(__ballot_sync(0xffffffffu, (v[1] >> 28) != 0u)) << 32);
    unsigned long long todo_hi = __ballot_sync(0xffffffffu, (v[2] >> 28) != 0u) |
                                 (static_cast<unsigned long long>(__ballot_sync(0xffffffffu, (v[3] >> 28) != 0u)) << 32);
    while (todo_lo | todo_hi) {
      int l = -1;  // position within the 128 rows
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int f = -1;
        if (todo_lo) {
          f = __ffsll(static_cast<long long>(todo_lo)) - 1;
          todo_lo &= todo_lo - 1;
        } else if (todo_hi) {
          f = 64 + __ffsll(static_cast<long long>(todo_hi)) - 1;
          todo_hi &= todo_hi - 1;
        }
        if (q == sub) l = f;
      }
      const int src = l < 0 ? 0 : (l & 31), gsel = l < 0 ? 0 : (l >> 5);
      const uint32_t w0 = __shfl_sync(0xffffffffu, v[0], src), w1 = __shfl_sync(0xffffffffu, v[1], src),
                     w2 = __shfl_sync(0xffffffffu, v[2], src), w3 = __shfl_sync(0xffffffffu, v[3], src);
      const uint32_t vv = gsel == 0 ? w0 : gsel == 1 ? w1 : gsel == 2 ? w2 : w3;
      const int64_t row = base + (l < 0 ? 0 : l);
      const int code = l < 0 ? 0 : static_cast<int>(vv >> 28);
      const int c1 = static_cast<int>(vv & 0x0fffffffu);
      if (code == 1 && li == 0) {
        p.nb[row] = c1;
        const unsigned long long idx = atomicAdd(p.flag_count, 1ull);
        p.flag_rows[idx] = static_cast<int32_t>(row);
      }
      const bool work = code >= 2;
      int cs[4] = {-1, -1, -1, -1};
      if (work) {
        const int4 rec = cand[row];
        cs[0] = c1;
        cs[1] = rec.x;
        cs[2] = code >= 3 ? rec.y : -1;
        cs[3] = code >= 4 ? rec.z : -1;
      }
      double ss = 0.0, dt[4] = {0.0, 0.0, 0.0, 0.0};
      if (work && vec) {  // 16-byte loads: four elements per lane and step
        const float* xr = p.X + row * d;
        for (int e = 4 * li; e < d; e += 32) {
          const float4 xv = *reinterpret_cast<const float4*>(xr + e);
          const double x0 = xv.x, x1 = xv.y, x2 = xv.z, x3 = xv.w;
          ss = fma(x0, x0, ss);
          ss = fma(x1, x1, ss);
          ss = fma(x2, x2, ss);
          ss = fma(x3, x3, ss);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (cs[j] >= 0) {
              const double* y = sums + static_cast<int64_t>(cs[j]) * d + e;
              const double2 a0 = *reinterpret_cast<const double2*>(y), a1 = *reinterpret_cast<const double2*>(y + 2);
              dt[j] = fma(a0.x, x0, dt[j]);
              dt[j] = fma(a0.y, x1, dt[j]);
              dt[j] = fma(a1.x, x2, dt[j]);
              dt[j] = fma(a1.y, x3, dt[j]);
            }
        }
      } else if (work) {
        for (int e = li; e < d; e += 8) {
          const double x = xval(p, row * d + e);
          ss = fma(x, x, ss);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (cs[j] >= 0) dt[j] = fma(sums[static_cast<int64_t>(cs[j]) * d + e], x, dt[j]);
        }
      }
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, off);
#pragma unroll
        for (int j = 0; j < 4; ++j) dt[j] += __shfl_xor_sync(0xffffffffu, dt[j], off);
      }
      if (li == 0 && work) {
        const double nrm = sqrt(ss);
        double best = 0.0;
        int arg = -1;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = cs[j];
          if (c < 0) continue;
          const double m = COS ? cos_foreign(p.nk[c], dt[j] / nrm) : sq_foreign(ss, p.stats[p.k + c], p.nk[c], dt[j]);
          if (arg < 0 || m < best || (m == best && c < arg)) {
            best = m;
            arg = c;
          }
        }
        p.nb[row] = arg;
        ++resolved;
      }
    }
  }
  for (int off = 16; off > 0; off >>= 1) resolved += __shfl_xor_sync(0xffffffffu, resolved, off);
  if (lane == 0 && resolved) atomicAdd(counts + 1, resolved);
}

template <bool COS>
__global__ void __launch_bounds__(256) pair_kernel(ScoreParams p, const int2* __restrict__ pairs,
                                                   const unsigned long long* count) {
  if (*p.abort) return;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  pair_rows_body<COS>(p, pairs, count, p.stats + (COS ? p.k : 2 * p.k), warp, nwarps, threadIdx.x & 31);
}

// Refinement of the flagged rows (cooperative launch, small cluster tables) -> grid
// barrier -> exact pass over every row -> fixed-order total in the last CTA.
template <bool COS, typename T, int LPR, int CPL>
__global__ void __launch_bounds__(kExactThreads) exact_kernel(ScoreParams p, ExactArgs ea) {
  griddep_wait();  // (PDL) the scoring pass's neighbours and flags are visible
  extern __shared__ __align__(16) double esm[];  // [stage: K*d table][refine: warps * d rows]
  const bool abort = *p.abort != 0;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const double* sums = p.stats + (COS ? p.k : 2 * p.k);
  const double* ytab = sums;
  const int64_t tab = static_cast<int64_t>(p.k) * p.d;
  if (ea.stage) {
    for (int64_t e = threadIdx.x; e < tab; e += blockDim.x) esm[e] = __ldg(sums + e);
    __syncthreads();
    ytab = esm;
  }
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wib;
  const int64_t gnw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  if (ea.refine) {
    if (!abort) {
      refine_rows<COS>(p, esm + (ea.stage ? tab : 0) + static_cast<int64_t>(wib) * p.d, gw, gnw, lane,
                       ea.stage ? esm : nullptr);
      if (ea.ta.pair_count) pair_rows_body<COS>(p, ea.pairs, ea.ta.pair_count, ytab, gw, gnw, lane);
    }
    grid_barrier(ea.bar, ea.bar + 1);  // every refined neighbour is written
  }
  if (!abort) exact_units<COS, T, LPR, CPL>(p, ytab, ea.usum, ea.nunits, gw, gnw, lane, ea.order);
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ea.ta.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) unit_total(ea, p.n);
}

}  // namespace

void flag_all(fsil_context* c, const ScoreParams& p, int tile_rows) {
  flag_all_kernel<<<static_cast<unsigned>((p.n + 255) / 256), 256, 0, c->stream>>>(
      p.n, tile_rows, p.flag_rows, p.tile_flag, p.tile_sum, p.flag_count);
  FSIL_LAUNCHED(c);
}

// Flagged-row count is only known on the device: the tiled kernel is chosen when the
// cluster-mean table is large (each row would otherwise re-read all of it from L2);
// its grid covers every flagged row of the worst case the table size allows.
void refine(fsil_context* c, const ScoreParams& p) {
  if (static_cast<int64_t>(c->k) * c->d >= 64 * 1024) {
    const int grid = c->num_sms * 4;
    const size_t entries = static_cast<size_t>(2) * grid * kRT;
    if (c->refine_cnt.bytes < grid * sizeof(unsigned)) {
      c->refine_cnt.ensure(grid * sizeof(unsigned));
      FSIL_CUDA(cudaMemsetAsync(c->refine_cnt.p, 0, c->refine_cnt.bytes, c->stream));
    }
    c->refine_part.ensure(entries * (sizeof(double) + sizeof(int)));
    const RefineSplit rs{c->refine_part.as<double>(), reinterpret_cast<int*>(c->refine_part.as<double>() + entries),
                         c->refine_cnt.as<unsigned>()};
    if (c->metric == FSIL_COSINE) refine_tiled_kernel<true><<<grid, 256, 0, c->stream>>>(p, rs);
    else refine_tiled_kernel<false><<<grid, 256, 0, c->stream>>>(p, rs);
    FSIL_LAUNCHED(c);
    return;
  }
  // warps per block limited by the staged rows (fp64 x per warp)
  const size_t row_bytes = static_cast<size_t>(c->d) * sizeof(double);
  const int wpb = static_cast<int>(std::min<size_t>(8, c->smem_optin / row_bytes));
  if (wpb < 1) fail(FSIL_ERR_INVALID_ARGUMENT, "refinement: D too large for shared memory");
  const size_t smem = wpb * row_bytes;
  const int grid = c->num_sms * 32 / wpb;
  if (c->metric == FSIL_COSINE) {
    FSIL_CUDA(cudaFuncSetAttribute(refine_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    refine_kernel<true><<<grid, 32 * wpb, smem, c->stream>>>(p);
  } else {
    FSIL_CUDA(cudaFuncSetAttribute(refine_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    refine_kernel<false><<<grid, 32 * wpb, smem, c->stream>>>(p);
  }
  FSIL_LAUNCHED(c);
}

namespace {
TotalArgs total_args(fsil_context* c, const ScoreParams& p, int64_t ngroups, bool local) {
  c->group_sum.ensure(ngroups * sizeof(double));
  c->result.ensure(4 * sizeof(double));
  TotalArgs ta;
  ta.group_sum = c->group_sum.as<double>();
  ta.result = c->result.as<double>();
  ta.flag_count = p.flag_count;
  ta.exact_count = nullptr;
  ta.pair_count = nullptr;
  ta.ticket = reinterpret_cast<unsigned int*>(c->counters.as<int>() + 8);
  ta.hsum = local ? c->dsum : nullptr;
  ta.checks = c->checks.as<int64_t>();
  ta.missing = c->counters.as<int>() + 4;
  return ta;
}
}  // namespace

// refine + finalize_sum as one cooperative launch when the per-row refine
// applies (cluster table below the tiled kernel's threshold); false: not applicable.
bool post_fused(fsil_context* c, const ScoreParams& p, int64_t ntiles, int tile_rows, bool local) {
  if (static_cast<int64_t>(c->k) * c->d >= 64 * 1024) return false;
  size_t smem = 8 * static_cast<size_t>(c->d) * sizeof(double);
  if (smem > c->smem_optin) return false;
  const size_t table = static_cast<size_t>(c->k) * c->d * sizeof(double);
  bool stage = smem + table <= 64 * 1024;  // small tables: staged per block
  if (stage) smem += table;
  const int64_t ngroups = std::max<int64_t>((ntiles + kGroupTiles - 1) / kGroupTiles, 1);
  TotalArgs ta = total_args(c, p, ngroups, local);
  unsigned int* bar = reinterpret_cast<unsigned int*>(c->counters.as<int>() + 12);
  void* kern = c->metric == FSIL_COSINE ? reinterpret_cast<void*>(post_kernel<true>)
                                        : reinterpret_cast<void*>(post_kernel<false>);
  FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  FSIL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
  if (per_sm < 1) return false;
  const int grid = c->num_sms;  // co-resident (the grid barrier needs it); one block per SM keeps the barrier short
  ScoreParams pp = p;
  int64_t nt = ntiles;
  int tr = tile_rows;
  void* args[] = {&pp, &nt, &tr, &ta, &bar, &stage};
  // cooperative (co-resident grid for the grid barrier) and, on the hot chain, PDL
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = 256;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  FSIL_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
  FSIL_LAUNCHED(c);
  return true;
}

// The exact pass (tensor-core path): every row's a_i, b_i, s_i in fp64 from its own and
// nominated neighbour cluster, then the deterministic total.  With a small cluster table
// (the per-row refinement applies) the flagged rows are refined in the same cooperative
// launch before a grid barrier; otherwise the tiled refinement runs first as its own
// launch.  D even (the tensor-core path needs D % 4 == 0).
void exact_pass(fsil_context* c, const ScoreParams& p, bool local) {
  const bool cos = c->metric == FSIL_COSINE;
  const bool x64 = c->X64 != nullptr;
  const int64_t tab = static_cast<int64_t>(c->k) * c->d;
  const bool small = tab < 64 * 1024;
  const unsigned long long* pcount = c->pair_count.as<unsigned long long>();
  if (c->tc_thr) {  // threshold mode: rows with two to four candidate neighbours, rows with none
    const unsigned cgrid = static_cast<unsigned>(c->num_sms * 8);
    unsigned long long* counts = c->pair_count.as<unsigned long long>();
    if (cos) launch_pdl(c, thr_resolve_kernel<true>, cgrid, 256, 0, p, c->cand_rows.as<int4>(), counts);
    else launch_pdl(c, thr_resolve_kernel<false>, cgrid, 256, 0, p, c->cand_rows.as<int4>(), counts);
  }
  if (!small) {  // full refinements (tiled) and certified pairs as their own launches
    refine(c, p);
    const unsigned pgrid = static_cast<unsigned>(c->num_sms * 8);
    if (cos) pair_kernel<true><<<pgrid, 256, 0, c->stream>>>(p, c->pair_rows.as<int2>(), pcount);
    else pair_kernel<false><<<pgrid, 256, 0, c->stream>>>(p, c->pair_rows.as<int2>(), pcount);
    FSIL_LAUNCHED(c);
  }
  const size_t tab_bytes = static_cast<size_t>(tab) * sizeof(double);
  const size_t rows_bytes = small ? (kExactThreads / 32) * static_cast<size_t>(c->d) * sizeof(double) : 0;
  const bool stage = tab_bytes + rows_bytes <= std::min<size_t>(c->smem_optin, 200 * 1024);
  const size_t smem = (stage ? tab_bytes : 0) + rows_bytes;
  ExactArgs ea{};
  ea.nunits = (c->n + kUnitRows - 1) / kUnitRows;
  c->group_sum.ensure(std::max<int64_t>(ea.nunits, 1) * sizeof(double));
  ea.usum = c->group_sum.as<double>();
  ea.ta = total_args(c, p, 1, local);
  ea.ta.group_sum = nullptr;
  ea.ta.pair_count = pcount;  // zeroed by agg_init; written only by the tcgen05 top-3 epilogue
  ea.pairs = c->pair_rows.as<int2>();
  ea.bar = reinterpret_cast<unsigned int*>(c->counters.as<int>() + 12);
  ea.refine = small ? 1 : 0;
  ea.stage = stage ? 1 : 0;
  // label-sorted order (FSIL_EXACT_SORTED=1; wide rows, cluster table in global memory): a
  // warp's consecutive rows share their own cluster's fp64 sums in cache.  Measured at C5:
  // 47.0 ms against 43.8 ms in row order (the gathered rows cost more than the table reuse
  // saves), so row order stays the default.
  static const bool order_env = [] {
    const char* e = std::getenv("FSIL_EXACT_SORTED");
    return e && std::atoi(e) != 0;
  }();
  ea.order = (order_env && !stage && c->agg_path == 2 && c->d >= 256 && !x64) ? c->sort_vals.as<int32_t>() : nullptr;
  // lanes per row / pairs per lane: D = 2 LPR CPL for the common widths, else generic
  const int d = c->d;
  int lpr = 32, cpl = 0;
  if (!x64) {
    // (a row's 16-byte pairs: 8 lanes read a table row's 128-byte line conflict-free)
    if (d == 16) lpr = 4, cpl = 2;
    else if (d == 32) lpr = 4, cpl = 4;
    else if (d == 64) lpr = 8, cpl = 4;
    else if (d == 128) lpr = 8, cpl = 8;
    else if (d == 256) lpr = 16, cpl = 8;
    else if (d == 512) lpr = 32, cpl = 8;
    else if (d == 768) lpr = 32, cpl = 12;
  }
  // the double2 reads of the cluster sums need 16-byte rows: a global table at an 8-byte
  // offset (cosine with odd K) takes the generic kernel's scalar reads
  const double* sums = p.stats + (cos ? c->k : 2 * c->k);
  if (!stage && (reinterpret_cast<uintptr_t>(sums) & 15)) lpr = 32, cpl = 0;
  void* kern = nullptr;
#define FSIL_EXACT_K(T, L, C)                                                                             \
  if (!kern && (sizeof(T) == 8) == x64 && lpr == L && cpl == C)                                           \
    kern = cos ? reinterpret_cast<void*>(exact_kernel<true, T, L, C>) : reinterpret_cast<void*>(exact_kernel<false, T, L, C>);
  FSIL_EXACT_K(float, 4, 2) FSIL_EXACT_K(float, 4, 4) FSIL_EXACT_K(float, 8, 4) FSIL_EXACT_K(float, 8, 8)
  FSIL_EXACT_K(float, 16, 8) FSIL_EXACT_K(float, 32, 8) FSIL_EXACT_K(float, 32, 12) FSIL_EXACT_K(float, 32, 0)
  FSIL_EXACT_K(double, 32, 0)
#undef FSIL_EXACT_K
  if (!kern) fail(FSIL_ERR_INTERNAL, "no exact-pass kernel for this shape");
  FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  FSIL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kExactThreads, smem));
  if (per_sm < 1) fail(FSIL_ERR_INTERNAL, "exact pass does not fit on an SM");
  const int grid = c->num_sms * std::min(per_sm, 2);
  ScoreParams pp = p;
  void* args[] = {&pp, &ea};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = kExactThreads;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[na++].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
  if (small) {  // co-resident grid for the grid barrier
    at[na].id = cudaLaunchAttributeCooperative;
    at[na++].val.cooperative = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  FSIL_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
  FSIL_LAUNCHED(c);
}

void finalize_sum(fsil_context* c, const ScoreParams& p, int64_t ntiles, int tile_rows, bool local) {
  const int64_t ngroups = std::max<int64_t>((ntiles + kGroupTiles - 1) / kGroupTiles, 1);
  TotalArgs ta = total_args(c, p, ngroups, local);
  tile_group_kernel<<<static_cast<unsigned>(ngroups), 256, 0, c->stream>>>(p.tile_sum, p.tile_flag, p.s, ntiles,
                                                                         tile_rows, p.n, ta);
  FSIL_LAUNCHED(c);
}

}  // namespace fsil
