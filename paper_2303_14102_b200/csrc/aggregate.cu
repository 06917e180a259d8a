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
#include <cstdlib>
#include <type_traits>

#include "device_util.cuh"
#include "fsil_internal.cuh"
#include "sm100.cuh"

namespace fsil {
namespace {

constexpr int kPieceRows = 2048;
constexpr int kRingWarps = 12, kRingCtas = 1;  // row-ring aggregation: warps per CTA, CTAs per SM

// ---------------------------------------------------------------- path 1 ----
// Warp-per-row streaming with the (warp-uniform) label of each row: lanes hold
// dims l + 32i (i < DPL), and each warp owns private fp64 accumulators in shared
// memory -- sums[K][D] (a row's read-modify-write touches consecutive doubles:
// bank-conflict free), per-lane Psi partials [K][32] (sqeuclid) and counts [K].
// U rows per warp are prefetched (labels through lanes 0..U-1).  Cosine row norms
// for the U rows are formed with a transpose-reduce across the warp (fp64).
// Rows are assigned warp-interleaved in a fixed pattern and every reduction is in
// a fixed order: bit-identical results run to run.
// T: the input element type (float, or double for the fp64 front end).
template <bool COS, int DPL, typename T>
__device__ __forceinline__ void agg_warp_rows(const T* __restrict__ X, const int32_t* __restrict__ dense,
                                              int64_t n, int d, int64_t row_offset, int64_t base, int64_t GW,
                                              bool checked, double* wsum, double* wpsi, double* wcnt,
                                              int64_t* checks, float& amax) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  const int64_t rl = base + (lane & (U - 1)) * GW;
  const int lab_l = (lane < U && (!checked || rl < n)) ? __ldg(dense + rl) : 0;
  T v[U][DPL];
  {
    const int64_t stride = GW * static_cast<int64_t>(d);
    const T* ptr = X + base * d + lane;
#pragma unroll
    for (int u = 0; u < U; ++u, ptr += stride) {
      const bool rv = !checked || base + u * GW < n;
#pragma unroll
      for (int i = 0; i < DPL; ++i)
        v[u][i] = (rv && (!checked || lane + 32 * i < d)) ? __ldcs(ptr + 32 * i) : T(0);
    }
  }
  double ss[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    ss[u] = 0.0;
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const double x = v[u][i];
      ss[u] = fma(x, x, ss[u]);
      amax = fmaxf(amax, fabsf(static_cast<float>(v[u][i])));
    }
  }
  double inv[U];
  if (COS) {
    // transpose-reduce: after three exchange steps lane L holds the partial of row
    // bit2(L) + 2*bit3(L) + 4*bit4(L) over 8 lanes; two xor steps finish all 32.
    double a4[4], a2[2], a1;
    const bool hi16 = lane & 16, hi8 = lane & 8, hi4 = lane & 4;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      a4[q] = (hi16 ? ss[q + 4] : ss[q]) + __shfl_xor_sync(0xffffffffu, hi16 ? ss[q] : ss[q + 4], 16);
#pragma unroll
    for (int q = 0; q < 2; ++q)
      a2[q] = (hi8 ? a4[q + 2] : a4[q]) + __shfl_xor_sync(0xffffffffu, hi8 ? a4[q] : a4[q + 2], 8);
    a1 = (hi4 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, hi4 ? a2[0] : a2[1], 4);
    a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
    a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
    // 1/||x||; 0 marks a zero row, NaN a non-finite one
    const double mine = a1 > 0.0 ? (a1 < INFINITY ? 1.0 / sqrt(a1) : NAN) : (a1 == 0.0 ? 0.0 : NAN);
#pragma unroll
    for (int u = 0; u < U; ++u)
      inv[u] = __shfl_sync(0xffffffffu, mine, (((u >> 2) & 1) << 4) | (((u >> 1) & 1) << 3) | ((u & 1) << 2));
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t r = base + u * GW;
    if (checked && r >= n) break;  // warp-uniform
    const int lab = __shfl_sync(0xffffffffu, lab_l, u);
    const bool bad = COS ? !(inv[u] == inv[u]) : __any_sync(0xffffffffu, !isfinite(ss[u]));
    if (bad) {  // rare: locate the non-finite element (dataset.cpp:35-37)
#pragma unroll
      for (int i = 0; i < DPL; ++i) {
        const int l = lane + 32 * i;
        if (l < d && !isfinite(v[u][i])) atomic_min_i64(checks, (row_offset + r) * d + l);
      }
    }
    if (COS && inv[u] == 0.0) {  // zero row (cos.cpp:119-123): reported, not accumulated
      if (lane == 0) atomic_min_i64(checks + 1, row_offset + r);
      continue;
    }
    double* ys = wsum + static_cast<int64_t>(lab) * d + lane;
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      if (!checked || lane + 32 * i < d)
        ys[32 * i] = COS ? fma(static_cast<double>(v[u][i]), inv[u], ys[32 * i]) : ys[32 * i] + static_cast<double>(v[u][i]);
    }
    if (!COS) wpsi[lab * 32 + lane] += ss[u];
    if (lane == 0) wcnt[lab] += 1.0;
  }
}

template <bool COS, int DPL, typename T>
__global__ void __launch_bounds__(256) agg_warp_kernel(
    const T* __restrict__ X, const int32_t* __restrict__ dense, int64_t n, int d,
    int64_t row_offset, int k, double* __restrict__ partials, int64_t* checks, float* xmax) {
  constexpr int U = 8;
  extern __shared__ double sm[];
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Sw = k * d + (COS ? 0 : k * 32) + k;  // per-warp doubles
  for (int j = threadIdx.x; j < warps * Sw; j += blockDim.x) sm[j] = 0.0;
  __syncthreads();
  double* wsum = sm + warp * Sw;                      // [k][d]
  double* wpsi = wsum + static_cast<int64_t>(k) * d;  // [k][32] (sqeuclid)
  double* wcnt = wpsi + (COS ? 0 : k * 32);           // [k]
  const int64_t GW = static_cast<int64_t>(gridDim.x) * warps;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * warps + warp;
  const bool full_d = d == 32 * DPL;
  float amax = 0.f;
  int64_t base = gw;
  if (full_d)  // unchecked fast path over complete groups of U rows
    for (; base + (U - 1) * GW < n; base += U * GW)
      agg_warp_rows<COS, DPL, T>(X, dense, n, d, row_offset, base, GW, false, wsum, wpsi, wcnt, checks, amax);
  for (; base < n; base += U * GW)
    agg_warp_rows<COS, DPL, T>(X, dense, n, d, row_offset, base, GW, true, wsum, wpsi, wcnt, checks, amax);
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  if (lane == 0 && amax > 0.f) atomic_max_nonneg_f32(xmax, amax);
  __syncthreads();
  // fold warps (fixed order) into the block partial in StatsLayout order
  const int S = COS ? k * (d + 1) : k * (d + 2);
  for (int j = threadIdx.x; j < S; j += blockDim.x) {
    double acc = 0.0;
    if (j < k) {
      for (int w = 0; w < warps; ++w) acc += sm[w * Sw + (COS ? k * d : k * d + k * 32) + j];
    } else if (!COS && j < 2 * k) {
      const int c = j - k;
      for (int w = 0; w < warps; ++w)
        for (int l = 0; l < 32; ++l) acc += sm[w * Sw + k * d + c * 32 + l];
    } else {
      const int t = j - (COS ? k : 2 * k);
      for (int w = 0; w < warps; ++w) acc += sm[w * Sw + t];
    }
    partials[static_cast<int64_t>(blockIdx.x) * S + j] = acc;
  }
}

// Same accumulation as agg_warp_kernel, but X streams HBM -> shared memory with 1-D
// bulk TMA copies (cp.async.bulk, mbarrier completion) through an NS-stage ring, so
// the bytes in flight per SM no longer depend on registers.  One CTA per SM owns a
// contiguous row range; consumer warp w takes rows w, w+W, ... of every stage.
template <bool COS, int DPL, int NS>
__global__ void __launch_bounds__(16 * 32, 1) agg_stage_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ dense, int64_t n, int d,
    int64_t row_offset, int k, int64_t chunk, double* __restrict__ partials, int64_t* checks,
    float* xmax) {
  constexpr int U = 8;
  extern __shared__ __align__(16) uint8_t smraw[];
  const int W = (blockDim.x >> 5) - 1;  // consumer warps; warp W is the producer
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = U * W;                  // rows per stage
  const int Sw = k * d + (COS ? 0 : k * 32) + k;
  double* sm = reinterpret_cast<double*>(smraw);
  // bulk-copy destinations need 16-byte alignment (W * Sw may be odd)
  float* ring = reinterpret_cast<float*>(sm + ((static_cast<size_t>(W) * Sw + 1) & ~size_t(1)));
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(NS) * R * d);
  uint64_t* full = bars;
  uint64_t* empty = bars + NS;
  for (int j = threadIdx.x; j < W * Sw; j += blockDim.x) sm[j] = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      sm100::mbar_init(full + i, 1);
      sm100::mbar_init(empty + i, W);
    }
    sm100::fence_barrier_init();
  }
  __syncthreads();
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t r1 = min(n, r0 + chunk);
  const int nstages = r1 > r0 ? static_cast<int>((r1 - r0 + R - 1) / R) : 0;
  if (warp == W) {
    if (lane == 0) {
      for (int i = 0; i < nstages; ++i) {
        const int s = i % NS;
        sm100::mbar_wait(empty + s, ((i / NS) & 1) ^ 1);
        const int64_t a = r0 + static_cast<int64_t>(i) * R;
        const int64_t nr = r1 - a < R ? r1 - a : static_cast<int64_t>(R);
        const uint32_t bytes = static_cast<uint32_t>(nr * d * 4);
        sm100::mbar_arrive_expect_tx(full + s, bytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                sm100::smem_u32(ring + static_cast<size_t>(s) * R * d)),
            "l"(X + a * d), "r"(bytes), "r"(sm100::smem_u32(full + s))
            : "memory");
      }
    }
    return;
  }
  double* wsum = sm + warp * Sw;
  double* wpsi = wsum + static_cast<int64_t>(k) * d;
  int* wcnt = reinterpret_cast<int*>(wpsi + (COS ? 0 : k * 32));  // [k] int counts
  const bool full_d = d == 32 * DPL;
  float amax = 0.f;
  for (int i = 0; i < nstages; ++i) {
    const int s = i % NS;
    sm100::mbar_wait(full + s, (i / NS) & 1);
    const int64_t a = r0 + static_cast<int64_t>(i) * R;
    const float* st = ring + static_cast<size_t>(s) * R * d;
    const bool full_stage = full_d && a + R <= r1;
    const int lab_l = (lane < U && a + lane * W + warp < r1) ? __ldg(dense + a + lane * W + warp) : 0;
    float v[U][DPL];
    if (full_stage) {
      const float* sp = st + warp * d + lane;
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < DPL; ++q) v[u][q] = sp[u * W * d + 32 * q];
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int lr = u * W + warp;
        const bool rv = a + lr < r1;
#pragma unroll
        for (int q = 0; q < DPL; ++q) {
          const int l = lane + 32 * q;
          v[u][q] = (rv && l < d) ? st[lr * d + l] : 0.f;
        }
      }
    }
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(empty + s);  // stage consumed into registers
    double ss[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ss[u] = 0.0;
#pragma unroll
      for (int q = 0; q < DPL; ++q) {
        const double x = v[u][q];
        ss[u] = fma(x, x, ss[u]);
        amax = fmaxf(amax, fabsf(v[u][q]));
      }
    }
    double inv[U];
    bool odd = false;  // any non-finite or (cosine) zero row in this group
    if (COS) {
      double a4[4], a2[2], a1;
      const bool hi16 = lane & 16, hi8 = lane & 8, hi4 = lane & 4;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        a4[q] = (hi16 ? ss[q + 4] : ss[q]) + __shfl_xor_sync(0xffffffffu, hi16 ? ss[q] : ss[q + 4], 16);
#pragma unroll
      for (int q = 0; q < 2; ++q)
        a2[q] = (hi8 ? a4[q + 2] : a4[q]) + __shfl_xor_sync(0xffffffffu, hi8 ? a4[q] : a4[q + 2], 8);
      a1 = (hi4 ? a2[1] : a2[0]) + __shfl_xor_sync(0xffffffffu, hi4 ? a2[0] : a2[1], 4);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
      const bool ok = a1 > 0.0 && a1 < INFINITY;
      const double mine = ok ? 1.0 / sqrt(a1) : 0.0;
      odd = __any_sync(0xffffffffu, !ok);
#pragma unroll
      for (int u = 0; u < U; ++u)
        inv[u] = __shfl_sync(0xffffffffu, mine, (((u >> 2) & 1) << 4) | (((u >> 1) & 1) << 3) | ((u & 1) << 2));
    } else {
      bool bad = false;
#pragma unroll
      for (int u = 0; u < U; ++u) bad = bad || !isfinite(ss[u]);
      odd = __any_sync(0xffffffffu, bad);
    }
    if (full_stage && !odd) {
      // ---- fast path: 8 valid rows, no checks.  Groups of four rows with distinct
      // labels (warp-uniform test) issue all their shared-memory loads before any
      // store, so the read-modify-writes overlap instead of serialising on a possible
      // alias; a group with a repeated label goes row by row.
      if (lane < U) atomicAdd(wcnt + lab_l, 1);
#pragma unroll
      for (int g = 0; g < U; g += 4) {
        int lab[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) lab[u] = __shfl_sync(0xffffffffu, lab_l, g + u);
        const bool distinct = lab[0] != lab[1] && lab[0] != lab[2] && lab[0] != lab[3] && lab[1] != lab[2] &&
                              lab[1] != lab[3] && lab[2] != lab[3];
        if (distinct) {
          double base[4][DPL], pb[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double* ys = wsum + lab[u] * d + lane;
#pragma unroll
            for (int q = 0; q < DPL; ++q) base[u][q] = ys[32 * q];
            if (!COS) pb[u] = wpsi[lab[u] * 32 + lane];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            double* ys = wsum + lab[u] * d + lane;
#pragma unroll
            for (int q = 0; q < DPL; ++q)
              ys[32 * q] = COS ? fma(static_cast<double>(v[g + u][q]), inv[g + u], base[u][q])
                               : base[u][q] + static_cast<double>(v[g + u][q]);
            if (!COS) wpsi[lab[u] * 32 + lane] = pb[u] + ss[g + u];
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            double* ys = wsum + lab[u] * d + lane;
#pragma unroll
            for (int q = 0; q < DPL; ++q)
              ys[32 * q] = COS ? fma(static_cast<double>(v[g + u][q]), inv[g + u], ys[32 * q])
                               : ys[32 * q] + static_cast<double>(v[g + u][q]);
            if (!COS) wpsi[lab[u] * 32 + lane] += ss[g + u];
          }
        }
      }
      continue;
    }
    // ---- general path (partial stage, non-finite or zero rows)
    double tot[U];
    if (COS) {
#pragma unroll
      for (int u = 0; u < U; ++u) tot[u] = inv[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = a + u * W + warp;
      if (r >= r1) break;  // warp-uniform
      const int lab = __shfl_sync(0xffffffffu, lab_l, u);
      double rs = ss[u];
      if (COS) {
        for (int off = 16; off > 0; off >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, off);
      }
      const bool bad = __any_sync(0xffffffffu, !isfinite(COS ? rs : ss[u]));
      if (bad) {  // locate the non-finite element (dataset.cpp:35-37)
#pragma unroll
        for (int q = 0; q < DPL; ++q) {
          const int l = lane + 32 * q;
          if (l < d && !isfinite(v[u][q])) atomic_min_i64(checks, (row_offset + r) * d + l);
        }
      }
      if (COS && rs == 0.0) {  // zero row (cos.cpp:119-123): reported, not accumulated
        if (lane == 0) atomic_min_i64(checks + 1, row_offset + r);
        continue;
      }
      const double sc = COS ? (isfinite(rs) ? 1.0 / sqrt(rs) : 0.0) : 1.0;
      double* ys = wsum + lab * d + lane;
#pragma unroll
      for (int q = 0; q < DPL; ++q)
        if (lane + 32 * q < d)
          ys[32 * q] = COS ? fma(static_cast<double>(v[u][q]), sc, ys[32 * q]) : ys[32 * q] + static_cast<double>(v[u][q]);
      if (!COS) wpsi[lab * 32 + lane] += ss[u];
      if (lane == 0) atomicAdd(wcnt + lab, 1);
    }
    (void)tot;
  }
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  if (lane == 0 && amax > 0.f) atomic_max_nonneg_f32(xmax, amax);
  // named barrier over the W consumer warps (the producer has returned)
  asm volatile("bar.sync 1, %0;\n" ::"r"(W * 32) : "memory");
  const int S = COS ? k * (d + 1) : k * (d + 2);
  for (int j = threadIdx.x; j < S; j += W * 32) {
    double acc = 0.0;
    if (j < k) {
      for (int w = 0; w < W; ++w)
        acc += static_cast<double>(reinterpret_cast<const int*>(sm + w * Sw + (COS ? k * d : k * d + k * 32))[j]);
    } else if (!COS && j < 2 * k) {
      const int c = j - k;
      for (int w = 0; w < W; ++w)
        for (int l = 0; l < 32; ++l) acc += sm[w * Sw + k * d + c * 32 + l];
    } else {
      const int t = j - (COS ? k : 2 * k);
      for (int w = 0; w < W; ++w) acc += sm[w * Sw + t];
    }
    partials[static_cast<int64_t>(blockIdx.x) * S + j] = acc;
  }
}

// Two-phase batched aggregation (D in {16, 32, 64, 128}, K*(D+2) small).  Every
// warp streams its own batches of 32 contiguous rows (one bulk copy each, double
// buffered per warp, no producer warp and no CTA-wide barrier) and
//   phase A  one lane per row: the row's fp64 ||x||^2 (rotated 16-byte chunks, so the
//            eight lanes of a shared-memory wavefront hit distinct banks), max|x|, the
//            finite / zero-norm checks, the count, and the row's scale (cosine
//            1/||x||; squared Euclidean the Psi contribution ||x||^2);
//   phase B  one lane per pair of dimensions: eight rows' contributions formed in
//            registers first, then eight read-modify-writes of the warp-private fp64
//            accumulators [K][D (+Psi, pad)].
// Compared with agg_stage (lanes own dimensions throughout) the per-row norm needs no
// cross-lane transpose-reduce or broadcast, and the label arrives by one shuffle.
// Rows go to warps in a fixed pattern and every sum has a fixed order: bit-identical
// results run to run.  Replaces the same reference code as agg_stage
// (squared_euclidean.cpp:37-54, cosine.cpp:39-61, cos.cpp:119-123, dataset.cpp:35-37).
template <int D, bool COS, int BR>
struct BatchCfg {
  static constexpr int NCH = D / 4;           // 16-byte chunks per row
  static constexpr int LPR = 32 / BR;         // phase-A lanes per row
  static constexpr int DX = COS ? D : D + 2;  // accumulated doubles per cluster: sums (+ Psi, pad)
  static constexpr int NP = DX / 2;           // double pairs per cluster
  static constexpr int PPL = (NP + 31) / 32;  // pairs per lane
  static constexpr int SLOT = BR * D;         // floats per batch slot
};

// batch rows: 16 (two phase-A lanes per row, more warps fit) unless D is small
__host__ __device__ inline int batch_rows(int d) { return d >= 64 ? 16 : 32; }

__host__ __device__ inline size_t batch_warp_bytes(int k, int d, bool cos) {
  const size_t dx = cos ? d : d + 2;
  const size_t br = batch_rows(d);
  return static_cast<size_t>(k) * dx * 8 + ((static_cast<size_t>(k) * 4 + 15) & ~size_t(15)) + br * 8 +
         2 * br * d * 4 + 16;
}

template <bool COS, int D, int BR>
__global__ void __launch_bounds__(16 * 32, 1) agg_batch_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ dense, int64_t n, int64_t row_offset, int k,
    double* __restrict__ partials, int64_t* checks, float* xmax, double* __restrict__ xi_out) {
  using C = BatchCfg<D, COS, BR>;
  extern __shared__ __align__(16) uint8_t smraw[];
  const int W = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int accw = k * C::DX;                          // doubles per warp accumulator
  const int cntw = ((k * 4 + 15) & ~15) / 4;           // ints per warp count array (16B multiple)
  double* acc = reinterpret_cast<double*>(smraw);      // [W][K][DX]
  int* cnt = reinterpret_cast<int*>(acc + static_cast<size_t>(W) * accw);  // [W][cntw]
  double* wv_all = reinterpret_cast<double*>(cnt + static_cast<size_t>(W) * cntw);  // [W][BR]
  float* slots = reinterpret_cast<float*>(wv_all + W * BR);                 // [W][2][SLOT]
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + static_cast<size_t>(W) * 2 * C::SLOT);  // [W][2]
  for (int j = threadIdx.x; j < W * accw; j += blockDim.x) acc[j] = 0.0;
  for (int j = threadIdx.x; j < W * cntw; j += blockDim.x) cnt[j] = 0;
  if (threadIdx.x < 2 * W) sm100::mbar_init(bars + threadIdx.x, 1);
  sm100::fence_barrier_init();
  __syncthreads();
  griddep_wait();  // (PDL) the set-up above overlaps the predecessor's tail

  double* wacc = acc + static_cast<size_t>(warp) * accw;
  int* wcnt = cnt + warp * cntw;
  double* wv = wv_all + warp * BR;
  float* wslot = slots + static_cast<size_t>(warp) * 2 * C::SLOT;
  uint64_t* wbar = bars + 2 * warp;
  const int64_t nb = (n + BR - 1) / BR;
  const int64_t G = static_cast<int64_t>(gridDim.x) * W;
  const int64_t g = static_cast<int64_t>(blockIdx.x) * W + warp;
  auto issue = [&](int64_t b, int s) {
    if (lane == 0) {
      const int64_t r0 = b * BR;
      const int64_t rows = n - r0 < BR ? n - r0 : BR;
      const uint32_t bytes = static_cast<uint32_t>(rows * D * 4);
      sm100::mbar_arrive_expect_tx(wbar + s, bytes);
      sm100::bulk_load(wslot + s * C::SLOT, X + r0 * D, bytes, wbar + s);
    }
  };
  if (g < nb) issue(g, 0);
  if (g + G < nb) issue(g + G, 1);

  const int rl = lane % BR, half = lane / BR;  // phase A: row, part of the row
  float amax = 0.f;
  int j = 0;
  for (int64_t b = g; b < nb; b += G, ++j) {
    const int s = j & 1;
    const int64_t r0 = b * BR;
    const int rows = static_cast<int>(n - r0 < BR ? n - r0 : BR);
    const bool rv = rl < rows;
    const int lab = rv ? __ldg(dense + r0 + rl) : 0;  // lanes rl and rl + BR hold the same row
    sm100::mbar_wait(wbar + s, (j >> 1) & 1);
    const float* sl = wslot + s * C::SLOT;

    // ---- phase A: LPR lanes per row
    double ss;
    {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (rv) {
        const float4* rp = reinterpret_cast<const float4*>(sl + rl * D);
#pragma unroll
        for (int i = 0; i < C::NCH / C::LPR; ++i) {
          const float4 f = rp[(i * C::LPR + half + rl) & (C::NCH - 1)];
          s0 = fma(static_cast<double>(f.x), static_cast<double>(f.x), s0);
          s1 = fma(static_cast<double>(f.y), static_cast<double>(f.y), s1);
          s2 = fma(static_cast<double>(f.z), static_cast<double>(f.z), s2);
          s3 = fma(static_cast<double>(f.w), static_cast<double>(f.w), s3);
          amax = fmaxf(amax, fmaxf(fabsf(f.x), fabsf(f.y)));
          amax = fmaxf(amax, fmaxf(fabsf(f.z), fabsf(f.w)));
        }
      }
      ss = (s0 + s1) + (s2 + s3);
      if (C::LPR == 2) ss += __shfl_xor_sync(0xffffffffu, ss, 16);
    }
    if (rv && half == 0) {
      const int64_t row = row_offset + r0 + rl;
      if (!isfinite(ss)) {  // rare: the first non-finite element of the row (dataset.cpp:35-37)
        for (int l = 0; l < D; ++l)
          if (!isfinite(sl[rl * D + l])) {
            atomic_min_i64(checks, row * D + l);
            break;
          }
      } else if (COS && ss == 0.0) {  // zero row (cos.cpp:119-123): reported
        atomic_min_i64(checks + 1, row);
      }
      wv[rl] = COS ? (ss > 0.0 && ss < INFINITY ? 1.0 / sqrt(ss) : 0.0) : ss;
      xi_out[r0 + rl] = ss;  // ||x||^2 for the scoring pass (fp64, from the exact squares)
      atomicAdd(wcnt + lab, 1);
    }
    __syncwarp();

    // ---- phase B: lane = pairs of dimensions (the Psi pair after the sums); eight
    // rows' contributions in registers, then their read-modify-writes in row order
    auto rows8 = [&](int rb, bool checked) {
      double2 p[8][C::PPL];
      int L[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = (rb + u) & (BR - 1);
        L[u] = __shfl_sync(0xffffffffu, lab, r);
        const double v = wv[r];
        const float* xr = sl + r * D;
#pragma unroll
        for (int q = 0; q < C::PPL; ++q) {
          const int pi = lane + 32 * q;
          if (pi < D / 2) {
            const float2 x = *reinterpret_cast<const float2*>(xr + 2 * pi);
            p[u][q] = COS ? make_double2(static_cast<double>(x.x) * v, static_cast<double>(x.y) * v)
                          : make_double2(static_cast<double>(x.x), static_cast<double>(x.y));
          } else {
            p[u][q] = make_double2(COS ? 0.0 : v, 0.0);  // squared Euclidean: (Psi, pad)
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (checked && rb + u >= rows) break;  // warp-uniform
#pragma unroll
        for (int q = 0; q < C::PPL; ++q) {
          const int pi = lane + 32 * q;
          if (pi < C::NP) {
            double2* a = reinterpret_cast<double2*>(wacc + L[u] * C::DX + 2 * pi);
            double2 t = *a;
            t.x += p[u][q].x;
            t.y += p[u][q].y;
            *a = t;
          }
        }
      }
    };
    if (rows == BR) {
#pragma unroll 1
      for (int rb = 0; rb < BR; rb += 8) rows8(rb, false);
    } else {
#pragma unroll 1
      for (int rb = 0; rb < rows; rb += 8) rows8(rb, true);
    }
    __syncwarp();  // every lane has read slot s
    if (b + 2 * G < nb) issue(b + 2 * G, s);
  }
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  if (lane == 0 && amax > 0.f) atomic_max_nonneg_f32(xmax, amax);
  __syncthreads();
  // fold the warps (fixed order) into this block's partial, StatsLayout order
  const int S = COS ? k * (D + 1) : k * (D + 2);
  for (int jj = threadIdx.x; jj < S; jj += blockDim.x) {
    double a = 0.0;
    if (jj < k) {
      for (int w = 0; w < W; ++w) a += static_cast<double>(cnt[w * cntw + jj]);
    } else if (!COS && jj < 2 * k) {
      const int c = jj - k;
      for (int w = 0; w < W; ++w) a += acc[static_cast<size_t>(w) * accw + c * C::DX + D];
    } else {
      const int t = jj - (COS ? k : 2 * k);
      const int c = t / D, l = t - c * D;
      for (int w = 0; w < W; ++w) a += acc[static_cast<size_t>(w) * accw + c * C::DX + l];
    }
    partials[static_cast<int64_t>(blockIdx.x) * S + jj] = a;
  }
}


// Sum of block partials per element: 8 fixed strided chains + fixed tree.
__global__ void __launch_bounds__(256) fold_partials_kernel(const double* __restrict__ partials,
                                                            int nblocks, int64_t S,
                                                            double* __restrict__ stats) {
  griddep_wait();
  __shared__ double sm[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  double acc = 0.0;
  if (j < S)
    for (int b0 = ty; b0 < nblocks; b0 += 64) {  // 8 loads in flight, then the same ordered adds
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = b0 + 8 * u < nblocks ? partials[static_cast<int64_t>(b0 + 8 * u) * S + j] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
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
template <bool COS, int VEC, int CPL, typename T>
__global__ void __launch_bounds__(256) agg_piece_kernel(
    const T* __restrict__ X, const int32_t* __restrict__ rows, int64_t n, int d,
    int64_t row_offset, int k, int lpr, const int64_t* __restrict__ seg_begin,
    const int64_t* __restrict__ seg_end, const int64_t* __restrict__ piece_start,
    double* __restrict__ piece_out, int64_t* checks, float* xmax, double* __restrict__ xi_out) {
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
  // U row groups per step: their index loads, then their row loads, are issued together (the
  // walk is a chain of two dependent loads per row otherwise -- latency-bound); the rows are
  // still accumulated one after the other, so every sum keeps its order.
  constexpr int U = CPL == 1 ? 4 : 1;  // (wider lanes: the row registers would spill)
  for (int64_t base0 = b0; base0 < b1; base0 += U * rpw) {
    int64_t ru[U];
    bool validu[U];
    T vu[U][CPL][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t pos = base0 + u * rpw + sub;  // warp-uniform trip count
      validu[u] = pos < b1;
      ru[u] = validu[u] ? rows[pos] : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int ch = li + q * lpr;
        if constexpr (VEC == 4) {  // float input only
          float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
          if (validu[u] && ch < nchunks) t = ldg_stream(reinterpret_cast<const float4*>(X + ru[u] * d) + ch);
          vu[u][q][0] = t.x; vu[u][q][1] = t.y; vu[u][q][2] = t.z; vu[u][q][3] = t.w;
        } else {
          vu[u][q][0] = (validu[u] && ch < nchunks) ? __ldg(X + ru[u] * d + ch) : T(0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
    if (base0 + u * rpw >= b1) break;  // (warp-uniform: groups past the piece's end)
    const bool valid = validu[u];
    const int64_t r = ru[u];
    T (&v)[CPL][VEC] = vu[u];
    double ss = 0.0;
    bool finite = true;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const double x = v[q][e];
        ss += x * x;
        finite = finite && isfinite(v[q][e]);
        amax = fmaxf(amax, fabsf(static_cast<float>(v[q][e])));
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
      if (valid && li == 0 && xi_out) xi_out[r] = ss;  // exact ||x||^2 for the scoring pass (cosine)
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

// ---------------------------------------------------------------- path 2 ----
// Hand-written stable counting sort of the rows by dense label (no library sort):
//   count   : G warp-chunks of L consecutive rows; each warp histograms its chunk in
//             shared memory (atomics; match_any groups equal labels when K is small) -> hist[c][g]
//   offsets : per label, an exclusive scan over the chunks (a row of chunk g lands
//             after every row of chunks < g with the same label) + the label's total
//   starts  : one block scans the K totals -> segment bounds, pieces per cluster and
//             their exclusive scan (the piece table)
//   scatter : each warp walks its chunk again in row order; a row's slot is its label's
//             running counter + its rank among equal labels in the 32-row group
// Rows of a label keep ascending row order, so every piece sum below is a fixed
// left-to-right order: bit-identical results run to run.
__global__ void __launch_bounds__(128) label_count_kernel(const int32_t* __restrict__ dense, int64_t n,
                                                          int64_t L, int G, int k, int32_t* __restrict__ hist) {
  extern __shared__ int32_t hsh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + w;
  int32_t* h = hsh + static_cast<size_t>(w) * k;
  for (int c = lane; c < k; c += 32) h[c] = 0;
  __syncwarp();
  if (g >= G) return;
  const int64_t b0 = static_cast<int64_t>(g) * L, b1 = min(n, b0 + L);
  constexpr int U = 4;  // 32-row groups whose labels are in flight together
  for (int64_t base = b0; base < b1; base += 32 * U) {
    int lab[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      lab[u] = i < b1 ? __ldg(dense + i) : -1;
    }
    if (k >= 64) {  // equal labels in a 32-row group are rare: shared-memory atomics
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (lab[u] >= 0) atomicAdd(h + lab[u], 1);
    } else {  // few labels: one add per distinct label of the group
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned peers = __match_any_sync(0xffffffffu, lab[u]);
        if (lab[u] >= 0 && lane == __ffs(peers) - 1) h[lab[u]] += __popc(peers);
        __syncwarp();
      }
    }
  }
  __syncwarp();
  for (int c = lane; c < k; c += 32) hist[static_cast<size_t>(c) * G + g] = h[c];
}

// block c: exclusive scan of hist[c][0..G) in place; totals[c] = the label's row count
__global__ void __launch_bounds__(256) label_offsets_kernel(int32_t* __restrict__ hist, int G, int64_t* totals) {
  __shared__ int32_t ws[8];
  const int c = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* h = hist + static_cast<size_t>(c) * G;
  int32_t carry = 0;
  for (int base = 0; base < G; base += 256) {
    const int j = base + threadIdx.x;
    const int32_t v = j < G ? h[j] : 0;
    int32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    int32_t wpre = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      wpre += q < w ? ws[q] : 0;
      tot += ws[q];
    }
    if (j < G) h[j] = carry + wpre + x - v;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[c] = carry;
}

// one block: segment bounds from the totals, pieces per cluster and the piece table
__global__ void __launch_bounds__(1024) label_starts_kernel(const int64_t* __restrict__ totals, int k,
                                                            int64_t* seg_begin, int64_t* seg_end,
                                                            int64_t* piece_start) {
  __shared__ int64_t ws[2][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int64_t carry_r = 0, carry_p = 0;
  for (int base = 0; base < k + 1; base += blockDim.x) {
    const int c = base + threadIdx.x;
    const int64_t t = c < k ? totals[c] : 0;
    const int64_t pc = (t + kPieceRows - 1) / kPieceRows;
    int64_t xr = t, xp = pc;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t yr = __shfl_up_sync(0xffffffffu, xr, off), yp = __shfl_up_sync(0xffffffffu, xp, off);
      if (lane >= off) {
        xr += yr;
        xp += yp;
      }
    }
    if (lane == 31) {
      ws[0][w] = xr;
      ws[1][w] = xp;
    }
    __syncthreads();
    int64_t pr = 0, pp = 0, tr = 0, tp = 0;
    for (int q = 0; q < nw; ++q) {
      pr += q < w ? ws[0][q] : 0;
      pp += q < w ? ws[1][q] : 0;
      tr += ws[0][q];
      tp += ws[1][q];
    }
    if (c <= k) {
      const int64_t begin = carry_r + pr + xr - t;
      if (c < k) {
        seg_begin[c] = begin;
        seg_end[c] = begin + t;
      }
      piece_start[c] = carry_p + pp + xp - pc;
    }
    carry_r += tr;
    carry_p += tp;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(128) label_scatter_kernel(const int32_t* __restrict__ dense, int64_t n,
                                                            int64_t L, int G, int k,
                                                            const int32_t* __restrict__ hist,
                                                            const int64_t* __restrict__ seg_begin,
                                                            int32_t* __restrict__ sorted_rows) {
  extern __shared__ int32_t hsh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + w;
  if (g >= G) return;
  int32_t* cnt = hsh + static_cast<size_t>(w) * k;  // next free slot of each label
  for (int c = lane; c < k; c += 32)
    cnt[c] = static_cast<int32_t>(seg_begin[c]) + hist[static_cast<size_t>(c) * G + g];
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  const int64_t b0 = static_cast<int64_t>(g) * L, b1 = min(n, b0 + L);
  constexpr int U = 4;
  for (int64_t base = b0; base < b1; base += 32 * U) {
    int lab[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      lab[u] = i < b1 ? __ldg(dense + i) : -1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {  // groups in row order: the sort stays stable
      const bool ok = lab[u] >= 0;
      const unsigned peers = __match_any_sync(0xffffffffu, lab[u]);
      if (ok) sorted_rows[cnt[lab[u]] + __popc(peers & lt)] = static_cast<int32_t>(base + u * 32 + lane);
      __syncwarp();
      if (ok && lane == __ffs(peers) - 1) cnt[lab[u]] += __popc(peers);
      __syncwarp();
    }
  }
}

// Pieces with the rows staged by bulk copies (fp32 rows of 16-byte multiples): each
// warp keeps R slots of rpw = 32 / lpr gathered rows in flight in its own shared-memory
// ring (one mbarrier per slot; lanes 0..rpw-1 each copy their row of the slot), so the
// row loads of a piece overlap instead of one row load per sub-group at a time.  The
// per-row arithmetic and the piece layout are agg_piece_kernel's.
template <bool COS, int CPL>
__global__ void __launch_bounds__(kRingWarps * 32, kRingCtas) agg_piece_ring_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ rows, int64_t n, int d,
    int64_t row_offset, int k, int lpr, int R, const int64_t* __restrict__ seg_begin,
    const int64_t* __restrict__ seg_end, const int64_t* __restrict__ piece_start,
    double* __restrict__ piece_out, int64_t* checks, float* xmax, double* __restrict__ xi_out) {
  extern __shared__ __align__(128) uint8_t rsh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int64_t p0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int rpw = 32 / lpr;
  const int row_bytes = d * 4;
  const int slot_bytes = rpw * row_bytes;
  uint8_t* ring = rsh + static_cast<size_t>(w) * R * slot_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rsh + static_cast<size_t>(nw) * R * slot_bytes) + w * R;
  // the gathered row ids of each slot (written by fill, read by the consumers: no global
  // load on the per-row critical path)
  int32_t* slot_rows = reinterpret_cast<int32_t*>(reinterpret_cast<uint64_t*>(rsh + static_cast<size_t>(nw) * R * slot_bytes) + nw * R) +
                       w * R * rpw;
  const int64_t total = piece_start[k];
  if (lane == 0)
    for (int s = 0; s < R; ++s) sm100::mbar_init(bars + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  int cs = 0;         // consumer slot
  uint32_t cph = 0;   // its phase parity
  int fs = 0;         // next slot to fill (ring order; runs R uses ahead of cs)
  for (int64_t p = p0; p < total; p += nwarps) {
    int lo = 0, hi = k - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (piece_start[mid] <= p) lo = mid;
      else hi = mid - 1;
    }
    const int c = lo;
    const int64_t b0 = seg_begin[c] + (p - piece_start[c]) * kPieceRows;
    const int64_t b1 = min(seg_end[c], b0 + kPieceRows);
    const int iters = static_cast<int>((b1 - b0 + rpw - 1) / rpw);
    // slot s <- the rows of iteration it (lanes 0..rpw-1 one row each; lane 0 arms the tx)
    auto fill = [&](int it, int s) {
      const int64_t pos = b0 + static_cast<int64_t>(it) * rpw + lane;
      const int nrows = static_cast<int>(min(static_cast<int64_t>(rpw), b1 - (b0 + static_cast<int64_t>(it) * rpw)));
      if (lane == 0) sm100::mbar_arrive_expect_tx(bars + s, nrows * row_bytes);
      if (lane < nrows) {
        const int32_t r = __ldg(rows + pos);
        slot_rows[s * rpw + lane] = r;
        sm100::bulk_load(ring + static_cast<size_t>(s) * slot_bytes + lane * row_bytes, X + static_cast<int64_t>(r) * d,
                         row_bytes, bars + s);
      }
    };
    for (int j = 0; j < R && j < iters; ++j) {
      fill(j, fs);
      if (++fs == R) fs = 0;
    }
    const int sub = lane / lpr, li = lane % lpr;
    const int nchunks = d >> 2;
    double acc[CPL][4];
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[q][e] = 0.0;
    double psi = 0.0, cnt = 0.0;
    float amax = 0.f;
    // Two slots (rows) per step: their norm reductions across the row's lanes (five
    // dependent shuffle steps, then a reciprocal square root for cosine) run side by
    // side and the per-step ring bookkeeping is paid once per two rows.  Rows are still
    // accumulated one after the other, so each lane's summation order is unchanged.
    constexpr int NR = CPL <= 3 ? 2 : 1;  // (wider rows: register budget)
    const bool full_lanes = nchunks == lpr * CPL;  // every lane's CPL chunks inside the row
    // one step of NR rows; FAST: all NR rows present and every chunk inside the row (no
    // per-element predicates, no zero fill)
    auto step = [&](int it, auto fast_tag) {
      constexpr bool FAST = decltype(fast_tag)::value;
      float v[NR][CPL][4];
      int64_t rr[NR];
      bool valid[NR];
#pragma unroll
      for (int h = 0; h < NR; ++h) {
        const int64_t pos = b0 + static_cast<int64_t>(it + h) * rpw + sub;
        valid[h] = FAST || (it + h < iters && pos < b1);
        rr[h] = 0;
        if (!FAST) {
#pragma unroll
          for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) v[h][q][e] = 0.f;
        }
        if (FAST || it + h < iters) {
          const int s = cs;
          sm100::mbar_wait(bars + s, cph);
          if (++cs == R) {
            cs = 0;
            cph ^= 1u;
          }
          const uint8_t* srow = ring + static_cast<size_t>(s) * slot_bytes + sub * row_bytes;
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            const int ch = li + q * lpr;
            if (FAST || (valid[h] && ch < nchunks)) {
              const float4 t = *reinterpret_cast<const float4*>(srow + ch * 16);
              v[h][q][0] = t.x; v[h][q][1] = t.y; v[h][q][2] = t.z; v[h][q][3] = t.w;
            }
          }
          if (valid[h]) rr[h] = slot_rows[s * rpw + sub];
        }
      }
      __syncwarp();  // every lane has read both slots: refill them
#pragma unroll
      for (int h = 0; h < NR; ++h)
        if (it + h + R < iters) {
          fill(it + h + R, fs);
          if (++fs == R) fs = 0;
        }
      // ||x||^2: four independent fp64 partials per lane (short dependency chains), a fixed
      // combination order, then the fixed xor-tree across the row's lanes
      double ss[NR];
      bool finite[NR];
#pragma unroll
      for (int h = 0; h < NR; ++h) {
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
        finite[h] = true;
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const double x = v[h][q][e];
            s4[e] = fma(x, x, s4[e]);
            if (!COS) finite[h] = finite[h] && isfinite(v[h][q][e]);
            amax = fmaxf(amax, fabsf(v[h][q][e]));
          }
        ss[h] = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        // cosine: squares of finite floats cannot overflow fp64, so a non-finite lane sum
        // flags the lane (one test per row instead of one per element)
        if (COS) finite[h] = isfinite(ss[h]);
      }
#pragma unroll
      for (int h = 0; h < NR; ++h)
        if (!finite[h]) {
#pragma unroll
          for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int l = (li + q * lpr) * 4 + e;
              if (l < d && !isfinite(v[h][q][e])) atomic_min_i64(checks, (row_offset + rr[h]) * d + l);
            }
        }
      if (COS) {
        for (int off = lpr >> 1; off > 0; off >>= 1) {
#pragma unroll
          for (int h = 0; h < NR; ++h) ss[h] += __shfl_xor_sync(0xffffffffu, ss[h], off, lpr);
        }
        double scale[NR];
#pragma unroll
        for (int h = 0; h < NR; ++h) {
          const bool ok = valid[h] && ss[h] != 0.0;
          scale[h] = ok ? 1.0 / sqrt(ss[h]) : 0.0;
          cnt += ok ? 1.0 : 0.0;
          if (valid[h] && li == 0) {
            if (xi_out) xi_out[rr[h]] = ss[h];
            if (ss[h] == 0.0) atomic_min_i64(checks + 1, row_offset + rr[h]);
          }
        }
#pragma unroll
        for (int h = 0; h < NR; ++h)  // row order (invalid rows add exact zeros)
#pragma unroll
          for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[q][e] += static_cast<double>(v[h][q][e]) * scale[h];
      } else {
#pragma unroll
        for (int h = 0; h < NR; ++h) {
          if (!FAST && !valid[h]) continue;
          psi += ss[h];
          cnt += 1.0;
#pragma unroll
          for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[q][e] += static_cast<double>(v[h][q][e]);
        }
      }
    };
    int it = 0;
    if (full_lanes)
      for (; it + NR <= iters; it += NR) step(it, std::true_type{});
    for (; it < iters; it += NR) step(it, std::false_type{});
    for (int off = 16; off >= lpr; off >>= 1) {
#pragma unroll
      for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[q][e] += __shfl_xor_sync(0xffffffffu, acc[q][e], off);
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
        for (int e = 0; e < 4; ++e) {
          const int l = (li + q * lpr) * 4 + e;
          if (l < d) sums[l] = acc[q][e];
        }
    }
  }
}

// Piece partials -> stats.  A block folds one cluster's 32-column slice: warp w sums the
// pieces p = w, w + 8, ... (lanes = columns: coalesced, independent loads), then the 8
// warp partials in a fixed order -- deterministic, and a large cluster's pieces are
// folded 8 x 32 wide instead of by one thread each.
__global__ void __launch_bounds__(256) fold_pieces_kernel(const double* __restrict__ piece_out,
                                                          const int64_t* __restrict__ piece_start, int k, int d,
                                                          bool cos, double* __restrict__ stats) {
  __shared__ double part[8][33];
  const int S1 = cos ? d + 1 : d + 2;
  const int nchunk = (S1 + 31) / 32;
  const int c = static_cast<int>(blockIdx.x / nchunk);
  const int j = static_cast<int>(blockIdx.x % nchunk) * 32 + (threadIdx.x & 31);
  const int w = threadIdx.x >> 5;
  double acc = 0.0;
  if (j < S1) {
    const int64_t p1 = piece_start[c + 1];
#pragma unroll 4
    for (int64_t p = piece_start[c] + w; p < p1; p += 8) acc += piece_out[p * S1 + j];
  }
  part[w][threadIdx.x & 31] = acc;
  __syncthreads();
  if (w == 0 && j < S1) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += part[q][threadIdx.x];
    if (j == 0) stats[c] = t;
    else if (!cos && j == 1) stats[k + c] = t;
    else stats[(cos ? k : 2 * k) + static_cast<int64_t>(c) * d + (j - (cos ? 1 : 2))] = t;
  }
}

// ---------------------------------------------------------------- derive ----
// Per-cluster constants of the scoring pass (fp32 operand copies + bounds).
__global__ void derive_kernel(const double* __restrict__ stats, int k, int d, int dp, bool cos,
                              float* mu32, float* p32, double* nk, float* bound) {
  griddep_wait();
  const int c = blockIdx.x;
  if (c >= k) {  // padding clusters up to the 32-multiple: zero operand rows (no memsets)
    for (int l = threadIdx.x; l < dp; l += blockDim.x) mu32[static_cast<int64_t>(c) * dp + l] = 0.f;
    if (threadIdx.x == 0) p32[c] = 0.f;
    return;
  }
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
    if (cos) p32[c] = 0.f;
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

// stats <- 0, validation word <- none, max|x| <- 0 (one launch instead of three copies)
__global__ void agg_init_kernel(double* stats, int64_t S, int64_t* checks, float* xmax, float* bound,
                                double* result, unsigned long long* flag_count,
                                unsigned long long* pair_count) {
  griddep_wait();
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < S; i += static_cast<int64_t>(gridDim.x) * blockDim.x) stats[i] = 0.0;
  if (i0 == 0) {
    checks[0] = kNone;
    checks[1] = kNone;
    *xmax = 0.f;
    for (int i = 0; i < 4; ++i) bound[i] = 0.f;  // derive's atomic maxima
    // the scoring phase's counters and partial result (no separate memsets per call)
    for (int i = 0; i < 4; ++i) result[i] = 0.0;
    *flag_count = 0ull;
    pair_count[0] = 0ull;
    pair_count[1] = 0ull;  // threshold mode's candidate records
  }
}

template <bool COS>
void launch_stage(fsil_context* c, int dpl, int warps, int64_t chunk, size_t smem, double* partials,
                  int64_t* checks, int ns) {
#define FSIL_AGG_STAGE(P)                                                                        \
  if (dpl == P) {                                                                                \
    auto kern = ns == 2 ? agg_stage_kernel<COS, P, 2> : agg_stage_kernel<COS, P, 3>;             \
    FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    kern<<<c->num_sms, (warps + 1) * 32, smem, c->stream>>>(c->X, c->dense.as<int32_t>(), c->n, c->d, \
                                             c->row_offset, c->k, chunk, partials, checks,       \
                                             c->xmax.as<float>());                               \
    FSIL_LAUNCHED(c);                                                                            \
    return;                                                                                      \
  }
  FSIL_AGG_STAGE(1) FSIL_AGG_STAGE(2) FSIL_AGG_STAGE(3) FSIL_AGG_STAGE(4)
#undef FSIL_AGG_STAGE
  fail(FSIL_ERR_INTERNAL, "no staged aggregation kernel for this shape");
}

template <bool COS>
void launch_batch(fsil_context* c, int warps, size_t smem, double* partials, int64_t* checks) {
#define FSIL_AGG_BATCH(DD)                                                                       \
  if (c->d == DD) {                                                                              \
    auto kern = agg_batch_kernel<COS, DD, DD >= 64 ? 16 : 32>;                                                       \
    FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    launch_pdl(c, kern, c->num_sms, warps * 32, smem, c->X, c->dense.as<int32_t>(), c->n,         \
               c->row_offset, c->k, partials, checks, c->xmax.as<float>(), c->xi_rows.as<double>()); \
    return;                                                                                      \
  }
  FSIL_AGG_BATCH(16) FSIL_AGG_BATCH(32) FSIL_AGG_BATCH(64) FSIL_AGG_BATCH(128)
#undef FSIL_AGG_BATCH
  fail(FSIL_ERR_INTERNAL, "no batched aggregation kernel for this shape");
}

template <bool COS, typename T>
void launch_warp(fsil_context* c, const T* X, int dpl, int grid, int threads, size_t smem, double* partials,
                 int64_t* checks) {
#define FSIL_AGG_WARP(P)                                                                         \
  if (dpl == P) {                                                                                \
    auto kern = agg_warp_kernel<COS, P, T>;                                                      \
    FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    kern<<<grid, threads, smem, c->stream>>>(X, c->dense.as<int32_t>(), c->n, c->d,             \
                                             c->row_offset, c->k, partials, checks,              \
                                             c->xmax.as<float>());                               \
    FSIL_LAUNCHED(c);                                                                            \
    return;                                                                                      \
  }
  FSIL_AGG_WARP(1) FSIL_AGG_WARP(2) FSIL_AGG_WARP(3) FSIL_AGG_WARP(4)
#undef FSIL_AGG_WARP
  fail(FSIL_ERR_INTERNAL, "no warp aggregation kernel for this shape");
}

template <bool COS, typename T>
void launch_pieces(fsil_context* c, const T* X, int vec, int cpl, int64_t max_pieces, int lpr,
                   const int32_t* rows, int64_t* seg_begin, int64_t* seg_end,
                   int64_t* piece_start, double* piece_out, int64_t* checks) {
  const unsigned grid = static_cast<unsigned>((max_pieces * 32 + 255) / 256);
#define FSIL_AGG_PIECE(V, C)                                                                     \
  if (vec == V && cpl == C) {                                                                    \
    agg_piece_kernel<COS, V, C, T><<<grid, 256, 0, c->stream>>>(                                 \
        X, rows, c->n, c->d, c->row_offset, c->k, lpr, seg_begin, seg_end, piece_start,          \
        piece_out, checks, c->xmax.as<float>(), c->xi_valid ? c->xi_rows.as<double>() : nullptr); \
    FSIL_LAUNCHED(c);                                                                            \
    return;                                                                                      \
  }
  if constexpr (sizeof(T) == 4) {
    FSIL_AGG_PIECE(4, 1) FSIL_AGG_PIECE(4, 2) FSIL_AGG_PIECE(4, 4) FSIL_AGG_PIECE(4, 8)
  }
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
  c->xmax.ensure(sizeof(float));
  c->xi_valid = false;
  c->bound.ensure(4 * sizeof(float));
  c->result.ensure(4 * sizeof(double));
  c->flag_count.ensure(sizeof(unsigned long long));
  c->pair_count.ensure(2 * sizeof(unsigned long long));
  launch_pdl(c, agg_init_kernel, static_cast<unsigned>(std::min<int64_t>((S + 255) / 256 + 1, 1024)), 256, 0, stats,
             S, checks, c->xmax.as<float>(), c->bound.as<float>(), c->result.as<double>(),
             c->flag_count.as<unsigned long long>(), c->pair_count.as<unsigned long long>());
  if (c->n == 0) {
    c->agg_path = 0;
    return;
  }
  // fp64 front end: the exact fp64 features (c->X64) feed the aggregation
  const bool x64 = c->X64 != nullptr;
  const int vec = (c->d % 4 == 0 && !x64) ? 4 : 1;
  const int lpr = pick_lpr(c->d, vec);
  const int chunks = (c->d + vec - 1) / vec;
  const int cpl = (chunks + lpr - 1) / lpr;

  // Path 1: warp-per-row with warp-private shared-memory accumulators, when at
  // least 8 such warps fit per SM (small K*D: C1, C2).
  const size_t budget = c->smem_optin ? c->smem_optin : 227 * 1024;
  const int dpl = (c->d + 31) / 32;
  const size_t per_warp = (static_cast<size_t>(c->k) * c->d + (cos ? 0 : c->k * 32) + c->k) * sizeof(double);
  int warps = 8;
  while (warps > 1 && warps * per_warp > budget) warps >>= 1;
  const size_t smem = warps * per_warp;
  const int blocks_per_sm = smem > 0 ? static_cast<int>(std::min<size_t>(228 * 1024 / (smem + 1024), 64 / warps)) : 0;
  // Path 1b: two-phase batches (D a power of two in 16..128); one CTA per SM with as
  // many warps (<= 16) as the per-warp accumulators and batch slots allow.
  static const bool batch_on = [] {
    const char* e = std::getenv("FSIL_AGG_BATCH");
    return !e || std::atoi(e) != 0;
  }();
  if (batch_on && !x64 && (c->d == 16 || c->d == 32 || c->d == 64 || c->d == 128)) {
    const size_t pw = batch_warp_bytes(c->k, c->d, cos);
    int W = 16;
    while (W > 4 && W * pw > budget) --W;
    if (W * pw <= budget) {
      c->agg_path = 3;
      c->xi_rows.ensure(static_cast<size_t>(c->n) * sizeof(double));
      c->xi_valid = true;
      const int grid = c->num_sms;
      c->partials.ensure(static_cast<size_t>(grid) * S * sizeof(double));
      if (cos) launch_batch<true>(c, W, W * pw, c->partials.as<double>(), checks);
      else launch_batch<false>(c, W, W * pw, c->partials.as<double>(), checks);
      launch_pdl(c, fold_partials_kernel, static_cast<unsigned>((S + 31) / 32), 256, 0, c->partials.as<double>(), grid,
                 S, stats);
      return;
    }
  }
  // Path 1a: bulk-TMA staged (needs 16-byte rows); one CTA per SM.
  if (dpl <= 4 && c->d % 4 == 0 && !x64) {
    // Consumer throughput bounds this kernel (measured at C2: T ~ 40 us + 632 us / W),
    // while the ring depth does not (NS = 2..6 alike): two stages, and as many
    // consumer warps (<= 15, one producer: 512 threads) as the private copies allow.
    // C2: W = 15 -> 89 us (W = 12, NS = 3: 95 us).
    int W = 15;
    const int NSs = 2;
    auto need = [&](int w) { return w * per_warp + 8 + static_cast<size_t>(NSs) * 8 * w * c->d * 4 + 64 + 16; };
    while (W > 4 && need(W) > budget) --W;
    if (need(W) <= budget && W >= 4) {
      c->agg_path = 1;
      const int64_t R = 8 * W;
      int64_t chunk = (c->n + c->num_sms - 1) / c->num_sms;
      chunk = (chunk + R - 1) / R * R;
      const int grid = c->num_sms;
      c->partials.ensure(static_cast<size_t>(grid) * S * sizeof(double));
      if (cos) launch_stage<true>(c, dpl, W, chunk, need(W), c->partials.as<double>(), checks, NSs);
      else launch_stage<false>(c, dpl, W, chunk, need(W), c->partials.as<double>(), checks, NSs);
      fold_partials_kernel<<<static_cast<unsigned>((S + 31) / 32), 256, 0, c->stream>>>(
          c->partials.as<double>(), grid, S, stats);
      FSIL_LAUNCHED(c);
      return;
    }
  }
  if (dpl <= 4 && smem <= budget && warps * blocks_per_sm >= 8) {
    c->agg_path = 1;
    const int64_t rows_per_block = static_cast<int64_t>(warps) * 8 * 4;
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>((c->n + rows_per_block - 1) / rows_per_block,
                             static_cast<int64_t>(c->num_sms) * blocks_per_sm)));
    c->partials.ensure(static_cast<size_t>(grid) * S * sizeof(double));
    if (x64) {
      if (cos) launch_warp<true>(c, c->X64, dpl, grid, warps * 32, smem, c->partials.as<double>(), checks);
      else launch_warp<false>(c, c->X64, dpl, grid, warps * 32, smem, c->partials.as<double>(), checks);
    } else {
      if (cos) launch_warp<true>(c, c->X, dpl, grid, warps * 32, smem, c->partials.as<double>(), checks);
      else launch_warp<false>(c, c->X, dpl, grid, warps * 32, smem, c->partials.as<double>(), checks);
    }
    fold_partials_kernel<<<static_cast<unsigned>((S + 31) / 32), 256, 0, c->stream>>>(
        c->partials.as<double>(), grid, S, stats);
    FSIL_LAUNCHED(c);
    return;
  }

  // Path 2: label-sorted segments.
  if (c->n >= (int64_t(1) << 31)) fail(FSIL_ERR_INVALID_ARGUMENT, "shard too large for the sorted aggregation path (2^31 rows)");
  // exact per-row ||x||^2 (fp64) for the scoring pass -- cosine only: there the sorted
  // pieces reduce each row's norm anyway, while for squared Euclidean the extra per-row
  // reduction and scattered 8-byte writes cost more than they save (measured: C3
  // aggregation 1.58 -> 3.74 ms, C4 5.7 -> 9.2 ms)
  if (!x64 && cos) {
    c->xi_rows.ensure(static_cast<size_t>(c->n) * sizeof(double));
    c->xi_valid = true;
  }
  const int cpl_max = vec == 4 ? 8 : 32;
  if (cpl > cpl_max)
    fail(FSIL_ERR_INVALID_ARGUMENT, "feature dimension too large for this build (D <= 1024)");
  c->agg_path = 2;
  c->seg_start.ensure((2 * static_cast<size_t>(c->k) + 2) * sizeof(int64_t));
  int64_t* seg_begin = c->seg_start.as<int64_t>();
  int64_t* seg_end = seg_begin + c->k + 1;
  c->piece_start.ensure((2 * static_cast<size_t>(c->k) + 4) * sizeof(int64_t));
  int64_t* ppc = c->piece_start.as<int64_t>();
  int64_t* piece_start = ppc + c->k + 2;
  c->sort_vals.ensure(c->n * sizeof(int32_t));
  // stable counting sort by dense label (hand-written, path 2 above): warps per block so
  // that the per-warp label counters fit shared memory
  int sw = 4;
  while (sw > 1 && static_cast<size_t>(sw) * c->k * sizeof(int32_t) > budget) sw >>= 1;
  static const bool cub_env = [] {
    const char* e = std::getenv("FSIL_AGG_CUB");
    return e && std::atoi(e) != 0;
  }();
  if (!cub_env && static_cast<size_t>(sw) * c->k * sizeof(int32_t) <= budget) {
    // warp-chunks: enough warps to keep the label loads in flight, while the K x G
    // histogram stays <= 16M entries
    const int64_t g_cap = std::max<int64_t>(static_cast<int64_t>(c->num_sms) * 16, (int64_t(16) << 20) / c->k);
    // (fewer, longer chunks -- runs of >= 32 rows per label and chunk, whole-sector scatter
    // writes -- measured slower at 1e8 rows: C4 aggregation 6.8 -> 7.5 ms)
    const int G = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((c->n + 1023) / 1024, g_cap)));
    const int64_t L = (c->n + G - 1) / G;
    const size_t hist_bytes = static_cast<size_t>(c->k) * G * sizeof(int32_t);
    c->sort_tmp.ensure(hist_bytes + static_cast<size_t>(c->k) * sizeof(int64_t) + 64);
    int32_t* hist = c->sort_tmp.as<int32_t>();
    int64_t* totals = reinterpret_cast<int64_t*>(c->sort_tmp.as<uint8_t>() + ((hist_bytes + 15) / 16) * 16);
    const unsigned sgrid = static_cast<unsigned>((G + sw - 1) / sw);
    const size_t ssm = static_cast<size_t>(sw) * c->k * sizeof(int32_t);
    if (ssm > 48 * 1024) {
      FSIL_CUDA(cudaFuncSetAttribute(label_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ssm)));
      FSIL_CUDA(cudaFuncSetAttribute(label_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ssm)));
    }
    label_count_kernel<<<sgrid, 32 * sw, ssm, c->stream>>>(c->dense.as<int32_t>(), c->n, L, G, c->k, hist);
    label_offsets_kernel<<<static_cast<unsigned>(c->k), 256, 0, c->stream>>>(hist, G, totals);
    label_starts_kernel<<<1, 1024, 0, c->stream>>>(totals, c->k, seg_begin, seg_end, piece_start);
    label_scatter_kernel<<<sgrid, 32 * sw, ssm, c->stream>>>(c->dense.as<int32_t>(), c->n, L, G, c->k, hist,
                                                             seg_begin, c->sort_vals.as<int32_t>());
    c->launches += 4;
  } else {
    // very large K: the library radix sort (cub) and scan
    const int n32 = static_cast<int>(c->n);
    c->iota.ensure(c->n * sizeof(int32_t));
    c->sort_keys.ensure(c->n * sizeof(int32_t));
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
    FSIL_CUDA(cudaMemsetAsync(seg_begin, 0, (2 * static_cast<size_t>(c->k) + 2) * sizeof(int64_t), c->stream));
    segment_bounds_kernel<<<static_cast<unsigned>((c->n + 255) / 256), 256, 0, c->stream>>>(
        c->sort_keys.as<int32_t>(), c->n, seg_begin, seg_end);
    FSIL_LAUNCHED(c);
    pieces_per_cluster_kernel<<<(c->k + 1 + 255) / 256, 256, 0, c->stream>>>(seg_begin, seg_end, c->k, ppc);
    FSIL_LAUNCHED(c);
    size_t scan_bytes = 0;
    FSIL_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, ppc, piece_start, c->k + 1, c->stream));
    if (scan_bytes > c->sort_tmp.bytes) c->sort_tmp.ensure(scan_bytes);
    FSIL_CUDA(cub::DeviceScan::ExclusiveSum(c->sort_tmp.p, scan_bytes, ppc, piece_start, c->k + 1, c->stream));
    c->launches += 1;
  }
  const int64_t max_pieces = c->n / kPieceRows + c->k + 1;
  const int S1 = cos ? c->d + 1 : c->d + 2;
  c->partials.ensure(static_cast<size_t>(max_pieces) * S1 * sizeof(double));
  const int cpl_t = cpl <= 1 ? 1 : cpl <= 2 ? 2 : cpl <= 4 ? 4 : cpl <= 8 ? 8 : cpl <= 16 ? 16 : 32;
  const int32_t* srows = c->sort_vals.as<int32_t>();
  static const bool ring_env = [] {
    const char* e = std::getenv("FSIL_AGG_RING");
    return !e || std::atoi(e) != 0;
  }();
  double* pout = c->partials.as<double>();
  if (x64) {
    if (cos) launch_pieces<true>(c, c->X64, vec, cpl_t, max_pieces, lpr, srows, seg_begin, seg_end, piece_start, pout, checks);
    else launch_pieces<false>(c, c->X64, vec, cpl_t, max_pieces, lpr, srows, seg_begin, seg_end, piece_start, pout, checks);
  } else if (vec == 4 && cpl <= 8 && c->d >= 256 && ring_env) {
    // wide rows (>= 1 KB): bulk-copy ring, R slots per warp, kRingCtas x kRingWarps
    // persistent warps per SM striding over the pieces.  The per-row arithmetic (fp64,
    // latency-bound) wants warps more than slots: random 3 KB row gathers reach HBM speed
    // with 16 rows in flight per SM (tools/gather_bench.cu).  Narrow rows keep
    // agg_piece_kernel (one bulk copy per small row costs more than it hides).
    const int rpw = 32 / lpr;
    const int slot = rpw * c->d * 4;
    const int W = kRingWarps;
    const size_t avail = std::min<size_t>(budget, 220 * 1024) / kRingCtas;
    const int R = static_cast<int>(std::max<size_t>(2, std::min<size_t>(16, avail / (static_cast<size_t>(W) * (slot + 8 + 4 * rpw)))));
    const size_t rsm = static_cast<size_t>(W) * R * (slot + 8 + 4 * rpw);
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(
        1, std::min<int64_t>((max_pieces + W - 1) / W, static_cast<int64_t>(kRingCtas) * c->num_sms)));
#define FSIL_AGG_RING(C)                                                                                   \
  if (cpl == C) {                                                                                          \
    auto kern = cos ? agg_piece_ring_kernel<true, C> : agg_piece_ring_kernel<false, C>;                    \
    FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rsm))); \
    kern<<<grid, 32 * W, rsm, c->stream>>>(c->X, srows, c->n, c->d, c->row_offset, c->k, lpr, R, seg_begin,  \
                                           seg_end, piece_start, pout, checks, c->xmax.as<float>(),          \
                                           c->xi_valid ? c->xi_rows.as<double>() : nullptr);                  \
    FSIL_LAUNCHED(c);                                                                                      \
  }
    FSIL_AGG_RING(2) else FSIL_AGG_RING(3) else FSIL_AGG_RING(4) else FSIL_AGG_RING(5) else FSIL_AGG_RING(6)
    else FSIL_AGG_RING(7) else FSIL_AGG_RING(8)
#undef FSIL_AGG_RING
  } else {
    if (cos) launch_pieces<true>(c, c->X, vec, cpl_t, max_pieces, lpr, srows, seg_begin, seg_end, piece_start, pout, checks);
    else launch_pieces<false>(c, c->X, vec, cpl_t, max_pieces, lpr, srows, seg_begin, seg_end, piece_start, pout, checks);
  }
  fold_pieces_kernel<<<static_cast<unsigned>(static_cast<int64_t>(c->k) * ((S1 + 31) / 32)), 256, 0, c->stream>>>(
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
  // (bound was zeroed by agg_init; padding rows are zeroed by their own blocks)
  launch_pdl(c, derive_kernel, static_cast<unsigned>(kpad), 128, 0, c->stats_buf.as<double>(), c->k, c->d,
             static_cast<int>(c->dp), cos, c->mu32.as<float>(), c->p32.as<float>(), c->nk.as<double>(),
             c->bound.as<float>());
}

}  // namespace fsil
