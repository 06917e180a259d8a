// score_ffma.cu -- K2: fused per-point scoring on the CUDA cores (small K).
//
// Replaces score_range + mean_dist_to_cluster + make_point_score
// (squared_euclidean.cpp:65-108, cosine.cpp:71-117, report.cpp:16-30) and the
// per-block part of finalize_report's sum (report.cpp:36-37).
//
// Per tile of 256 rows (128 threads, 2 rows per thread):
//   * X streams HBM -> shared memory with cp.async (double-buffered, padded
//     row stride so every thread's 128-bit row reads are bank-conflict free);
//   * fast pass: K fp32 dot products per row with packed FFMA2
//     (__ffma2_rn, even/odd partial sums), cluster means broadcast from smem;
//     clamped foreign means, top-2 with a rigorous fp32 error bound eps_row;
//   * the nominated neighbour is certain when best2 - best1 > 2 eps_row;
//     otherwise the row is appended to the refinement list (K4 re-evaluates
//     every cluster in fp64 with the reference's strict-< lowest-index rule);
//   * a_i and b_i are recomputed in fp64 with the reference formulas for the
//     own and nominated clusters, s_i assembled, and a fixed-order tile sum of
//     s_i written for the deterministic global mean.
#include <algorithm>

#include "score_common.cuh"

namespace fsil {
namespace {

constexpr int kThreads = 128;
constexpr int kRowsPerThread = 2;
constexpr int kTileRows = kThreads * kRowsPerThread;

template <int VEC>
__device__ __forceinline__ void load_tile(const ScoreParams& p, float* xs, int64_t tile) {
  const int64_t row0 = tile * kTileRows;
  if constexpr (VEC == 4) {
    const int cpr = p.dp >> 2;  // 16-byte chunks per row (dp == d here)
    const int step_row = kThreads / cpr, step_ch = kThreads % cpr;
    int row = threadIdx.x / cpr, ch = threadIdx.x % cpr;
    while (row < kTileRows) {
      const int64_t g = row0 + row;
      const bool valid = g < p.n;
      cp_async16(xs + row * p.xstride + ch * 4, p.X + (valid ? g : 0) * p.d + ch * 4, valid);
      ch += step_ch;
      row += step_row;
      if (ch >= cpr) {
        ch -= cpr;
        ++row;
      }
    }
  } else {
    const int step_row = kThreads / p.dp, step_ch = kThreads % p.dp;
    int row = threadIdx.x / p.dp, l = threadIdx.x % p.dp;
    while (row < kTileRows) {
      const int64_t g = row0 + row;
      const bool valid = g < p.n && l < p.d;
      cp_async4(xs + row * p.xstride + l, p.X + (valid ? g * p.d + l : 0), valid);
      l += step_ch;
      row += step_row;
      if (l >= p.dp) {
        l -= p.dp;
        ++row;
      }
    }
  }
  cp_async_commit();
}

template <int KB, bool COS, int VEC, bool MULTI>
__global__ void __launch_bounds__(kThreads) score_ffma_kernel(ScoreParams p, int64_t ntiles) {
  if (*p.abort) return;  // K speculation missed: the call is repeated
  extern __shared__ __align__(16) float smem[];
  // single-group case: Yt2[dp/2][KB] pairs {Y[k][l], Y[k][l+1]} (fp64) so that the
  // per-lane own/neighbour gathers of the fp64 epilogue all hit one smem row
  double2* yt2 = reinterpret_cast<double2*>(smem);
  float* mus = smem + (MULTI ? 0 : KB * p.dp * 2);      // [KB][dp]
  float* pks = mus + (MULTI ? 0 : KB * p.dp);           // [KB]
  float* xbuf = pks + (MULTI ? 0 : KB);                 // [nstage][kTileRows][xstride]
  __shared__ double wsum[kThreads / 32];
  const int tid = threadIdx.x;
  const int nstage = p.nstage;

  if constexpr (!MULTI) {
    for (int j = tid; j < KB * p.dp; j += kThreads) mus[j] = p.mu32[j];
    for (int j = tid; j < KB; j += kThreads) pks[j] = COS ? 0.f : p.p32[j];
    const double* sums = p.stats + (COS ? p.k : 2 * p.k);
    for (int j = tid; j < KB * (p.dp / 2); j += kThreads) {
      const int k = j % KB, l2 = j / KB;
      double2 v = make_double2(0.0, 0.0);
      if (k < p.k) {
        const int l = 2 * l2;
        if (l < p.d) v.x = sums[static_cast<int64_t>(k) * p.d + l];
        if (l + 1 < p.d) v.y = sums[static_cast<int64_t>(k) * p.d + l + 1];
      }
      yt2[j] = v;
    }
  }

  const float bmu = p.bound[0], bp = p.bound[1];
  const float gam = gamma_f32(p.dp + 6);
  const int nc = p.dp >> 2;
  const int ngroups = MULTI ? (p.k + KB - 1) / KB : 1;

  int64_t tile = blockIdx.x;
  int buf = 0;
  if (tile < ntiles) load_tile<VEC>(p, xbuf, tile);
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t next = tile + gridDim.x;
    float* xs = xbuf + buf * kTileRows * p.xstride;
    if (nstage == 2 && next < ntiles) {
      load_tile<VEC>(p, xbuf + (buf ^ 1) * kTileRows * p.xstride, next);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    const float* xr[kRowsPerThread];
    int own[kRowsPerThread];
    float xi[kRowsPerThread], inv[kRowsPerThread], best1[kRowsPerThread], best2[kRowsPerThread];
    int arg[kRowsPerThread];
#pragma unroll
    for (int r = 0; r < kRowsPerThread; ++r) {
      const int64_t row = tile * kTileRows + tid + r * kThreads;
      xr[r] = xs + (tid + r * kThreads) * p.xstride;
      own[r] = row < p.n ? p.dense[row] : -1;
      best1[r] = INFINITY;
      best2[r] = INFINITY;
      arg[r] = -1;
      xi[r] = 0.f;
      inv[r] = 0.f;
    }

    for (int g = 0; g < ngroups; ++g) {
      const int kbase = g * KB;
      // ---------------- fast pass: fp32 dots (packed FFMA2) ----------------
      float2 acc[kRowsPerThread][KB];
      float2 sq[kRowsPerThread];
#pragma unroll
      for (int r = 0; r < kRowsPerThread; ++r) {
        sq[r] = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < KB; ++j) acc[r][j] = make_float2(0.f, 0.f);
      }
      const float* mug = MULTI ? p.mu32 + static_cast<int64_t>(kbase) * p.dp : mus;
#pragma unroll 2
      for (int c = 0; c < nc; ++c) {
        float4 xv[kRowsPerThread];
#pragma unroll
        for (int r = 0; r < kRowsPerThread; ++r) {
          xv[r] = *reinterpret_cast<const float4*>(xr[r] + 4 * c);
          if (g == 0) {
            sq[r] = __ffma2_rn(make_float2(xv[r].x, xv[r].y), make_float2(xv[r].x, xv[r].y), sq[r]);
            sq[r] = __ffma2_rn(make_float2(xv[r].z, xv[r].w), make_float2(xv[r].z, xv[r].w), sq[r]);
          }
        }
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          const float4 m = MULTI ? __ldg(reinterpret_cast<const float4*>(mug + j * p.dp + 4 * c))
                                 : *reinterpret_cast<const float4*>(mug + j * p.dp + 4 * c);
#pragma unroll
          for (int r = 0; r < kRowsPerThread; ++r) {
            acc[r][j] = __ffma2_rn(make_float2(xv[r].x, xv[r].y), make_float2(m.x, m.y), acc[r][j]);
            acc[r][j] = __ffma2_rn(make_float2(xv[r].z, xv[r].w), make_float2(m.z, m.w), acc[r][j]);
          }
        }
      }
#pragma unroll
      for (int r = 0; r < kRowsPerThread; ++r) {
        if (g == 0) {
          xi[r] = sq[r].x + sq[r].y;
          if (COS) inv[r] = 1.0f / sqrtf(xi[r]);
        }
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          const int kk = kbase + j;
          if (kk < p.k && kk != own[r]) {
            const float dot = acc[r][j].x + acc[r][j].y;
            float m;
            if (COS) m = fminf(fmaxf(1.0f - dot * inv[r], 0.0f), 2.0f);
            else m = fmaxf((xi[r] + (MULTI ? __ldg(p.p32 + kk) : pks[j])) - 2.0f * dot, 0.0f);
            if (m < best1[r]) {
              best2[r] = best1[r];
              best1[r] = m;
              arg[r] = kk;
            } else if (m < best2[r]) {
              best2[r] = m;
            }
          }
        }
      }
    }

    // ---------------- epilogue ----------------
    int nbr[kRowsPerThread];
    bool flg[kRowsPerThread];
#pragma unroll
    for (int r = 0; r < kRowsPerThread; ++r) {
      const float eps = COS ? 1.01f * gam * (2.0f * bmu + 2.0f)
                            : 1.01f * gam * (xi[r] + bp + 4.0f * sqrtf(xi[r]) * bmu);
      flg[r] = !((best2[r] - best1[r]) > 2.0f * eps);
      nbr[r] = arg[r];
      if (nbr[r] < 0) {  // non-finite fast pass (overflowing features): provisional pick
        nbr[r] = own[r] == 0 ? 1 : 0;
        flg[r] = true;
      }
      if (own[r] < 0) {  // row past n: harmless in-range indices
        own[r] = 0;
        nbr[r] = 1;
      }
    }
    // fp64 a_i, b_i with the reference formulas: own and neighbour dots (+ ||x||^2)
    double ss[kRowsPerThread], co[kRowsPerThread], cb[kRowsPerThread];
#pragma unroll
    for (int r = 0; r < kRowsPerThread; ++r) ss[r] = co[r] = cb[r] = 0.0;
    if constexpr (!MULTI) {
#pragma unroll 2
      for (int c = 0; c < nc; ++c) {
#pragma unroll
        for (int r = 0; r < kRowsPerThread; ++r) {
          const float4 xv = *reinterpret_cast<const float4*>(xr[r] + 4 * c);
          const double2 yo0 = yt2[(2 * c) * KB + own[r]], yo1 = yt2[(2 * c + 1) * KB + own[r]];
          const double2 yb0 = yt2[(2 * c) * KB + nbr[r]], yb1 = yt2[(2 * c + 1) * KB + nbr[r]];
          const double x0 = xv.x, x1 = xv.y, x2 = xv.z, x3 = xv.w;
          ss[r] = fma(x0, x0, ss[r]); ss[r] = fma(x1, x1, ss[r]);
          ss[r] = fma(x2, x2, ss[r]); ss[r] = fma(x3, x3, ss[r]);
          co[r] = fma(yo0.x, x0, co[r]); co[r] = fma(yo0.y, x1, co[r]);
          co[r] = fma(yo1.x, x2, co[r]); co[r] = fma(yo1.y, x3, co[r]);
          cb[r] = fma(yb0.x, x0, cb[r]); cb[r] = fma(yb0.y, x1, cb[r]);
          cb[r] = fma(yb1.x, x2, cb[r]); cb[r] = fma(yb1.y, x3, cb[r]);
        }
      }
    } else {
      const double* sums = p.stats + (COS ? p.k : 2 * p.k);
#pragma unroll
      for (int r = 0; r < kRowsPerThread; ++r) {
        const double* yo = sums + static_cast<int64_t>(own[r]) * p.d;
        const double* yb = sums + static_cast<int64_t>(nbr[r]) * p.d;
        for (int l = 0; l < p.d; ++l) {
          const double v = xr[r][l];
          ss[r] = fma(v, v, ss[r]);
          co[r] = fma(__ldg(yo + l), v, co[r]);
          cb[r] = fma(__ldg(yb + l), v, cb[r]);
        }
      }
    }
    double s_thread = 0.0;
    bool any_flag = false;
#pragma unroll
    for (int r = 0; r < kRowsPerThread; ++r) {
      const int64_t row = tile * kTileRows + tid + r * kThreads;
      if (row >= p.n) continue;
      const double n_o = p.nk[own[r]], n_b = p.nk[nbr[r]];
      const bool singleton = n_o == 1.0;
      double a, b;
      if (COS) {
        const double nrm = sqrt(ss[r]);
        b = cos_foreign(n_b, cb[r] / nrm);
        a = singleton ? 0.0 : cos_own(n_o, co[r] / nrm);
      } else {
        b = sq_foreign(ss[r], p.stats[p.k + nbr[r]], n_b, cb[r]);
        a = singleton ? 0.0 : sq_own(ss[r], p.stats[p.k + own[r]], n_o, co[r]);
      }
      const double s = singleton ? 0.0 : assemble_score(a, b);
      p.s[row] = s;
      if (p.nb) p.nb[row] = nbr[r];
      if (p.own) p.own[row] = own[r];
      if (p.a) p.a[row] = a;
      if (p.b) p.b[row] = b;
      if (flg[r]) {
        const unsigned long long idx = atomicAdd(p.flag_count, 1ull);
        p.flag_rows[idx] = static_cast<int32_t>(row);
        any_flag = true;
      }
      s_thread += s;
    }
    // fixed-order tile sum of s_i
    for (int off = 16; off > 0; off >>= 1) s_thread += __shfl_xor_sync(0xffffffffu, s_thread, off);
    if ((tid & 31) == 0) wsum[tid >> 5] = s_thread;
    const int tile_flagged = __syncthreads_or(any_flag);
    if (tid == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) t += wsum[w];
      p.tile_sum[tile] = t;
      p.tile_flag[tile] = tile_flagged;
    }
    __syncthreads();  // xs and wsum are reused next iteration
    if (nstage == 2) buf ^= 1;
    else if (next < ntiles) load_tile<VEC>(p, xbuf, next);
  }
}

struct Launch {
  int kb;
  void* fn;
};

template <bool COS, int VEC>
void* pick_kernel(int kb) {
  switch (kb) {
    case 4: return reinterpret_cast<void*>(score_ffma_kernel<4, COS, VEC, false>);
    case 8: return reinterpret_cast<void*>(score_ffma_kernel<8, COS, VEC, false>);
    case 12: return reinterpret_cast<void*>(score_ffma_kernel<12, COS, VEC, false>);
    case 16: return reinterpret_cast<void*>(score_ffma_kernel<16, COS, VEC, false>);
    case 20: return reinterpret_cast<void*>(score_ffma_kernel<20, COS, VEC, false>);
    case 24: return reinterpret_cast<void*>(score_ffma_kernel<24, COS, VEC, false>);
    case 28: return reinterpret_cast<void*>(score_ffma_kernel<28, COS, VEC, false>);
    case 32: return reinterpret_cast<void*>(score_ffma_kernel<32, COS, VEC, false>);
    case -1: return reinterpret_cast<void*>(score_ffma_kernel<16, COS, VEC, true>);
  }
  return nullptr;
}

}  // namespace

int64_t ffma_tiles(int64_t n) { return (n + kTileRows - 1) / kTileRows; }

static size_t ffma_smem(const fsil_context* c, int* xstride_out, int nstage) {
  const int kb = c->k <= 32 ? std::max(4, ((c->k + 3) / 4) * 4) : -1;
  const int q = static_cast<int>(c->dp / 4);
  const int xstride = static_cast<int>(c->dp) + ((q % 2 == 0) ? 4 : 8);
  if (xstride_out) *xstride_out = xstride;
  const size_t mu_floats = kb > 0 ? static_cast<size_t>(kb) * c->dp * 3 + kb : 0;
  return (mu_floats + static_cast<size_t>(nstage) * kTileRows * xstride) * sizeof(float);
}

// Two stages in one CTA when two such CTAs still fit per SM, else single-stage
// CTAs (overlap then comes from the co-resident CTAs).
static int ffma_stages(const fsil_context* c) {
  const size_t sm_bytes = 228 * 1024;
  return ffma_smem(c, nullptr, 2) * 2 + 2048 <= sm_bytes ? 2 : 1;
}

bool ffma_supported(const fsil_context* c) { return ffma_smem(c, nullptr, 1) <= c->smem_optin; }

void score_ffma(fsil_context* c, const ScoreParams& base) {
  const bool cos = c->metric == FSIL_COSINE;
  const int vec = c->d % 4 == 0 ? 4 : 1;
  // K <= 32: cluster means resident in shared memory, one group.  Larger K:
  // groups of 16 clusters with means read through L1 (correct at any K; the
  // tensor-core kernel is the fast path there).
  const int kb = c->k <= 32 ? std::max(4, ((c->k + 3) / 4) * 4) : -1;
  ScoreParams p = base;
  // padded row stride: (xstride/4) odd -> conflict-free 128-bit row reads
  p.nstage = ffma_stages(c);
  const size_t smem = ffma_smem(c, &p.xstride, p.nstage);
  void* fn = cos ? (vec == 4 ? pick_kernel<true, 4>(kb) : pick_kernel<true, 1>(kb))
                 : (vec == 4 ? pick_kernel<false, 4>(kb) : pick_kernel<false, 1>(kb));
  if (smem > c->smem_optin)
    fail(FSIL_ERR_INVALID_ARGUMENT, "feature dimension too large for the FFMA scoring tile");
  FSIL_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  FSIL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem));
  per_sm = std::max(per_sm, 1);
  const int64_t ntiles = ffma_tiles(c->n);
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, int64_t(c->num_sms) * per_sm)));
  void* args[] = {&p, const_cast<int64_t*>(&ntiles)};
  FSIL_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, smem, c->stream));
  FSIL_LAUNCHED(c);
}

}  // namespace fsil
