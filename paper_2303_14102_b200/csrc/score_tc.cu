// score_tc.cu -- K3: per-point scoring on the 5th-generation tensor cores.
//
// Replaces score_range + mean_dist_to_cluster + make_point_score
// (squared_euclidean.cpp:65-108, cosine.cpp:71-117, report.cpp:16-30) when
// X . mu^T is a real contraction.  One persistent CTA per SM, warp-specialised:
//
//   warp 0      TMA producer: fp32 X boxes (128 rows x 32 cols, 128B swizzle) into a
//               staging ring; fp16 cluster-mean pieces B_hi/B_lo into the operand ring
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer (kind::f16, fp32 accum)
//   warps 2..5  epilogue (one TMEM lane = one row): clamped cluster means, top-2 with a
//               rigorous error bound, a_i/b_i/s_i from the tensor-core dots in fp64
//   warps 6..9  converters: x (fp32) -> x*2^-ex split into fp16 hi + lo in the UMMA
//               K-major SWIZZLE_128B layout, plus ||x||^2 (fp32 and fp64) per row
//
// Split precision ("fp16x3"): x~ = hx + lx, mu~ = hm + lm (exact to ~2^-22 after a
// global power-of-two scaling); dot = hx.hm + hx.lm + lx.hm, three MMAs per K step.
// Every row carries a certified bound on its dots; rows whose neighbour is not
// certain go to the fp64 argmin refinement (K4), rows whose a_i/b_i bound exceeds
// 5e-6 in s_i go to the exact own/neighbour recompute -- both in finalize.cu.
#include <algorithm>
#include <cmath>
#include <cuda_fp16.h>

#include "score_common.cuh"
#include "sm100.cuh"

namespace fsil {
namespace {

using namespace sm100;

constexpr int BM = 128;               // rows per tile = TMEM lanes
constexpr int BK = 64;                // fp16 K elements per chunk (one 128-byte swizzle row)
constexpr int kStgBytes = 2 * BM * 128;  // two fp32 boxes of 32 columns
constexpr int kABytes = BM * 128;        // one fp16 A piece (hi or lo)
constexpr int kThreads = 480;            // 15 warps
constexpr float kTau = 9e-6f;            // certified |ds_i| budget before exact a/b (bar: 1e-5)

__host__ __device__ constexpr int ncb_bn_pad(int kp) { return (kp + 3) & ~3; }

struct TcParams {
  ScoreParams p;
  int ncb, nkc;           // cluster blocks, K chunks
  float sx;               // 2^-ex: x -> x~
  float smul;             // 2^(ex+em): dot = acc * smul
  double smul64;
  const float* colbias;   // [ncb*BN]: sqeuclid p_k, cosine 0, padding +inf
  const float* munorm;    // [ncb*BN]: ||mu_k|| rounded up (per-cluster error bounds)
  const double4* clu;     // [K]: {n_k, 1/(n_k-1) (0 if singleton), Psi_k, 0}
  float cdot;             // relative dot bound coefficient
  float floor_coef;       // absolute-floor coefficient (times ||x||)
  float mu_max;           // max ||mu_k||
  float p_max;
  int2* exact_rows;       // rows needing the exact own/neighbour recompute
  unsigned long long* exact_count;
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

template <int BN>
struct TcCfg {
  static constexpr int kStg = BN <= 32 ? 4 : BN <= 64 ? 3 : 2;  // fp32 X staging stages
  static constexpr int kOps = 2;                                 // operand (A+B) stages
  static constexpr int kBBytes = BN * 128;
  static constexpr int kOpBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr size_t kRing = static_cast<size_t>(kStg) * kStgBytes + static_cast<size_t>(kOps) * kOpBytes;
};

template <int BN, bool COS>
__global__ void __launch_bounds__(kThreads, 1)
    score_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_bh,
                    const __grid_constant__ CUtensorMap tmap_bl, TcParams tp, int64_t ntiles) {
  using C = TcCfg<BN>;
  constexpr int NS = C::kStg, NO = C::kOps;
  // TS (BN <= 64): the two epilogue groups take alternate tiles, each with its own
  // pair of accumulator buffers, so consecutive tiles' epilogues overlap.  Otherwise
  // the groups split the column chunks of every tile.
  constexpr bool TS = BN <= 64;
  constexpr int NACC = TS ? 4 : 2;
  constexpr uint32_t kCols = NACC * 2 * BN;  // x {main, correction}
  constexpr uint32_t kTmemCols = (kCols <= 32) ? 32 : (kCols <= 64) ? 64 : (kCols <= 128) ? 128 : (kCols <= 256) ? 256 : 512;
  constexpr uint32_t kIdesc = idesc_f16_f32(BM, BN);
  const ScoreParams& p = tp.p;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = base;                     // [NS][kStgBytes]
  uint8_t* ops = stg + NS * kStgBytes;     // [NO][a_hi | a_lo | b_hi | b_lo]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ops + NO * C::kOpBytes);
  uint64_t* stg_full = bars;               // [NS]
  uint64_t* stg_empty = bars + 4;          // [NS]
  uint64_t* op_full = bars + 8;            // [NO]
  uint64_t* op_empty = bars + 10;          // [NO]
  uint64_t* acc_full = bars + 12;          // [NACC]
  uint64_t* acc_empty = bars + 16;         // [NACC]
  uint64_t* meta_full = bars + 20;         // [2]
  uint64_t* meta_empty = bars + 22;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  double* meta_xi = reinterpret_cast<double*>(bars + 26);   // [2][BM] ||x||^2 (fp64 of fp32 blocks)
  float* part = reinterpret_cast<float*>(meta_xi + 2 * BM);  // [2][4][BM] second-half partial top-2
  double* red = reinterpret_cast<double*>(part + 8 * BM);     // [2][4] tile-sum partials
  int* red_flag = reinterpret_cast<int*>(red + 8);            // [2][4]
  float* cb_s = reinterpret_cast<float*>(red + 12);           // [ncb*BN] column bias

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncb = tp.ncb, nkc = tp.nkc;
  for (int j = threadIdx.x; j < ncb * BN; j += blockDim.x) cb_s[j] = tp.colbias[j];

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(stg_full + i, 1);
      mbar_init(stg_empty + i, 4);
    }
    for (int i = 0; i < NO; ++i) {
      mbar_init(op_full + i, 1 + 4);
      mbar_init(op_empty + i, 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(acc_full + i, 1);
      mbar_init(acc_empty + i, TS ? 4 : 8);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(meta_full + i, 4);
      mbar_init(meta_empty + i, TS ? 4 : 8);
    }
    fence_barrier_init();
    prefetch_tmap(&tmap_x);
    prefetch_tmap(&tmap_bh);
    prefetch_tmap(&tmap_bl);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer: X
    if (lane == 0) {
      uint32_t n1 = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int row0 = static_cast<int>(t * BM);
        for (int cb = 0; cb < ncb; ++cb) {
          for (int kc = 0; kc < nkc; ++kc, ++n1) {
            const int s1 = n1 % NS;
            const int nbox = (kc * BK + 32 < p.d) ? 2 : 1;
            mbar_wait(stg_empty + s1, ((n1 / NS) & 1) ^ 1);
            mbar_arrive_expect_tx(stg_full + s1, nbox * BM * 128);
            for (int b = 0; b < nbox; ++b)
              tma_load_2d(stg + s1 * kStgBytes + b * BM * 128, &tmap_x, stg_full + s1, kc * BK + b * 32, row0);
          }
        }
      }
    }
  } else if (warp == 14) {
    // ------------------------------------------------------------ TMA producer: B pieces
    if (lane == 0) {
      uint32_t n2 = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int cb = 0; cb < ncb; ++cb) {
          for (int kc = 0; kc < nkc; ++kc, ++n2) {
            const int s2 = n2 % NO;
            uint8_t* op = ops + s2 * C::kOpBytes;
            mbar_wait(op_empty + s2, ((n2 / NO) & 1) ^ 1);
            mbar_arrive_expect_tx(op_full + s2, 2 * C::kBBytes);
            tma_load_2d(op + 2 * kABytes, &tmap_bh, op_full + s2, kc * BK, cb * BN);
            tma_load_2d(op + 2 * kABytes + C::kBBytes, &tmap_bl, op_full + s2, kc * BK, cb * BN);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t n2 = 0, na = 0, ng[2] = {0, 0}, nt = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
        for (int cb = 0; cb < ncb; ++cb, ++na) {
          int ab;
          uint32_t ph;
          if (TS) {
            const int g = nt & 1;
            ab = 2 * g + (ng[g] & 1);
            ph = (ng[g] >> 1) & 1;
            ++ng[g];
          } else {
            ab = na & 1;
            ph = (na >> 1) & 1;
          }
          mbar_wait(acc_empty + ab, ph ^ 1);
          tc_fence_after();
          const uint32_t d_main = tmem_base + ab * 2 * BN, d_corr = d_main + BN;
          for (int kc = 0; kc < nkc; ++kc, ++n2) {
            const int s2 = n2 % NO;
            mbar_wait(op_full + s2, (n2 / NO) & 1);
            tc_fence_after();
            const int rem = p.d - kc * BK;
            const int nks = rem >= BK ? 4 : (rem + 15) / 16;
            const uint32_t ah = smem_u32(ops + s2 * C::kOpBytes), al = ah + kABytes;
            const uint32_t bh = ah + 2 * kABytes, bl = bh + C::kBBytes;
            for (int ks = 0; ks < nks; ++ks) {
              const uint32_t off = ks * 32;
              const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
              // main term and the two correction terms accumulate separately: the
              // corrections are ~2^-10 of the main term, so their fp32 rounding is too
              mma_f16(d_main, desc_k_sw128(ah + off), desc_k_sw128(bh + off), kIdesc, acc0);
              mma_f16(d_corr, desc_k_sw128(ah + off), desc_k_sw128(bl + off), kIdesc, acc0);
              mma_f16(d_corr, desc_k_sw128(al + off), desc_k_sw128(bh + off), kIdesc, 1u);
            }
            mma_commit(op_empty + s2);  // operand stage free once these MMAs retire
          }
          mma_commit(acc_full + ab);    // accumulators ready for the epilogue
        }
      }
    }
  } else if (warp >= 10 && warp < 14) {
    // ------------------------------------------------------------ converters
    const int r = threadIdx.x - 10 * 32;  // row in tile, 0..127
    const int sw = r & 7;
    uint32_t n1 = 0, n2 = 0, nt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
      double xi = 0.0;
      for (int cb = 0; cb < ncb; ++cb) {
        for (int kc = 0; kc < nkc; ++kc, ++n1, ++n2) {
          const int s1 = n1 % NS, s2 = n2 % NO;
          mbar_wait(stg_full + s1, (n1 / NS) & 1);
          mbar_wait(op_empty + s2, ((n2 / NO) & 1) ^ 1);
          const uint8_t* srow = stg + s1 * kStgBytes + r * 128;
          uint8_t* hrow = ops + s2 * C::kOpBytes + r * 128;
          uint8_t* lrow = hrow + kABytes;
          const bool two = kc * BK + 32 < p.d;
#pragma unroll
          for (int j = 0; j < 8; ++j) {  // 8 fp16 A chunks of 16 bytes
            float4 f0 = make_float4(0.f, 0.f, 0.f, 0.f), f1 = f0;
            if (j < 4 || two) {
              const uint8_t* box = srow + (j >> 2) * (BM * 128);
              f0 = *reinterpret_cast<const float4*>(box + ((((2 * j) & 7) ^ sw) << 4));
              f1 = *reinterpret_cast<const float4*>(box + ((((2 * j + 1) & 7) ^ sw) << 4));
            }
            const float v[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
            if (cb == 0) {  // ||x||^2: fp32 blocks of 8 (error <= 8u each), fp64 across blocks
              float bs = 0.f;
#pragma unroll
              for (int e = 0; e < 8; ++e) bs = fmaf(v[e], v[e], bs);
              xi += static_cast<double>(bs);
            }
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float x0 = v[2 * e] * tp.sx, x1 = v[2 * e + 1] * tp.sx;
              const __half2 h = __floats2half2_rn(x0, x1);
              const float2 hf = __half22float2(h);
              const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
              hw[e] = *reinterpret_cast<const uint32_t*>(&h);
              lw[e] = *reinterpret_cast<const uint32_t*>(&l);
            }
            const int pos = (j ^ sw) << 4;
            *reinterpret_cast<uint4*>(hrow + pos) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(lrow + pos) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(op_full + s2);
            mbar_arrive(stg_empty + s1);
          }
        }
        if (cb == 0) {
          const int tb = nt & 1;
          mbar_wait(meta_empty + tb, ((nt >> 1) & 1) ^ 1);
          meta_xi[tb * BM + r] = xi;
          __syncwarp();
          if (lane == 0) mbar_arrive(meta_full + tb);
        }
      }
    }
  } else if (warp >= 2) {
    // ------------------------------------------------------------ epilogue (8 warps)
    const int quad = warp & 3;        // TMEM lane quadrant of this warp
    const int r = quad * 32 + lane;   // row in tile
    const int grp = (warp - 2) >> 2;  // epilogue group 0 / 1
    uint32_t na = 0, nt = 0, ng = 0;
    constexpr int NQ = BN / 32;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
      const int tb = nt & 1;
      if (TS && tb != grp) continue;  // the other group takes this tile
      const int64_t row = t * BM + r;
      const bool valid = row < p.n;
      const int own = valid ? p.dense[row] : -1;
      mbar_wait(meta_full + tb, (nt >> 1) & 1);
      const double xi64 = meta_xi[tb * BM + r];
      const float xi = static_cast<float>(xi64);
      const float xn = sqrtf(xi);
      // ranking key m' = m - rowc (row constant dropped, no clamp): sqeuclid
      // m = xi + p_k - 2 dot, cosine m = 1 - dot/||x||; dot = acc * smul
      const float rowm = COS ? -(tp.smul / xn) : -2.0f * tp.smul;
      float b1 = INFINITY, b2 = INFINITY, doto = NAN;
      int arg = -1;
      for (int cb = 0; cb < ncb; ++cb) {
        int ab;
        uint32_t ph;
        if (TS) {
          ab = 2 * grp + (ng & 1);
          ph = (ng >> 1) & 1;
          ++ng;
        } else {
          ab = na & 1;
          ph = (na >> 1) & 1;
          ++na;
        }
        mbar_wait(acc_full + ab, ph);
        tc_fence_after();
#pragma unroll 1
        for (int q = TS ? 0 : grp; q < NQ; q += TS ? 1 : 2) {
          float v[32], w[32];
          const uint32_t ta = tmem_base + ab * 2 * BN + q * 32 + (static_cast<uint32_t>(quad * 32) << 16);
          tmem_ld32(ta, v);
          tmem_ld32(ta + BN, w);
          const int k0 = cb * BN + q * 32;
          const float4* cb4 = reinterpret_cast<const float4*>(cb_s + k0);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 bias = cb4[j4];
            const float bj[4] = {bias.x, bias.y, bias.z, bias.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = 4 * j4 + e;
              const int k = k0 + j;
              const float acc = v[j] + w[j];
              float m = fmaf(acc, rowm, bj[e]);
              const bool is_own = k == own;
              doto = is_own ? acc : doto;
              m = is_own ? INFINITY : m;
              const bool lt = m < b1;  // strict: the lowest index keeps ties
              arg = lt ? k : arg;
              b2 = fminf(b2, fmaxf(b1, m));
              b1 = fminf(b1, m);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + ab);
      }
      if (!TS) {
        // ---- merge the two column halves (group 1 -> smem -> group 0)
        float* pt = part + tb * 4 * BM;  // double-buffered by tile parity
        if (grp == 1) {
          pt[0 * BM + r] = b1;
          pt[1 * BM + r] = b2;
          pt[2 * BM + r] = __int_as_float(arg);
          pt[3 * BM + r] = doto;
        }
        named_bar(1, 256);
        if (grp == 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(meta_empty + tb);
          continue;
        }
        const float c1 = pt[0 * BM + r], c2 = pt[1 * BM + r];
        const int a2 = __float_as_int(pt[2 * BM + r]);
        const float d2 = pt[3 * BM + r];
        const float nb1 = fminf(b1, c1);
        b2 = fminf(fminf(fmaxf(b1, c1), b2), c2);
        arg = (c1 < b1 || (c1 == b1 && a2 >= 0 && (arg < 0 || a2 < arg))) ? a2 : arg;
        b1 = nb1;
        doto = (doto == doto) ? doto : d2;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(meta_empty + tb);

      // ---- certification and a_i, b_i, s_i (no fp64 divisions: per-cluster
      // reciprocals precomputed, 1/||x|| and 1/max(a,b) by Newton steps in fp64)
      double s = 0.0;
      bool any = false;
      if (valid) {
        const float u = 5.9604645e-8f;
        const float rowc = COS ? 1.0f : xi;
        const float exi = 8.1f * u * xi;   // ||x||^2 error (fp32 blocks of 8)
        const float eps_dot = (tp.cdot * tp.mu_max + tp.floor_coef) * xn;  // any column
        const float eps_m = COS ? (eps_dot / xn + 3.0f * u * (fabsf(b1) + 1.0f) + exi / xi)
                                : (2.0f * eps_dot + 3.0f * u * (fabsf(b1) + tp.p_max + 2.0f * xn * tp.mu_max) + exi);
        int nb = arg;
        // neighbour certain: clear gap, and no tie through the clamps at 0 (and 2)
        const bool full = !((b2 - b1) > 2.0f * eps_m) || nb < 0 || !(rowc + b2 > eps_m) ||
                          (COS && !(rowc + b1 < 2.0f - eps_m));
        if (nb < 0) nb = own == 0 ? 1 : 0;
        const double4 co = tp.clu[own];  // n, 1/(n-1), Psi
        const bool singleton = co.x == 1.0;
        const double ed_b = (static_cast<double>(tp.cdot) * __ldg(tp.munorm + nb) + tp.floor_coef) * xn;
        const double ed_o = (static_cast<double>(tp.cdot) * __ldg(tp.munorm + own) + tp.floor_coef) * xn;
        const double dob = static_cast<double>(doto) * tp.smul64;
        const double mb = static_cast<double>(rowc) + static_cast<double>(b1);
        const double n_o = co.x, r_o = co.y, nr_o = n_o * r_o;
        double a, b, da, db;
        if (COS) {
          double rn = static_cast<double>(rsqrtf(xi));
          rn = rn * (1.5 - 0.5 * xi64 * rn * rn);
          rn = rn * (1.5 - 0.5 * xi64 * rn * rn);  // 1/||x|| to ~1e-16
          b = fmin(fmax(mb, 0.0), 2.0);
          a = singleton ? 0.0 : fmin(fmax((n_o - n_o * dob * rn) * r_o, 0.0), 2.0);
          db = ed_b * rn + 3.0 * u * (fabs(b1) + 1.0) + exi / xi;
          da = nr_o * (ed_o * rn + exi / xi);
        } else {
          b = fmax(mb, 0.0);
          a = singleton ? 0.0 : fmax((n_o * xi64 + co.z - 2.0 * n_o * dob) * r_o, 0.0);
          db = 2.0 * ed_b + 3.0 * u * (fabs(b1) + tp.p_max + 2.0 * xn * tp.mu_max) + exi;
          da = nr_o * (2.0 * ed_o + exi);
        }
        const double mx = fmax(a, b);
        if (!singleton && mx > 0.0) {  // assemble_score without a division
          double rm = static_cast<double>(__frcp_rn(static_cast<float>(mx)));
          rm = rm * (2.0 - mx * rm);
          rm = rm * (2.0 - mx * rm);
          s = a <= b ? 1.0 - a * rm : b * rm - 1.0;
        }
        const bool inexact = !singleton && !(mx > 2.0 * (da + db) && (da + db) <= static_cast<double>(kTau) * mx);
        p.s[row] = s;
        if (p.nb) p.nb[row] = nb;
        if (p.own) p.own[row] = own;
        if (p.a) p.a[row] = a;
        if (p.b) p.b[row] = b;
        if (full) {
          const unsigned long long idx = atomicAdd(p.flag_count, 1ull);
          p.flag_rows[idx] = static_cast<int32_t>(row);
          any = true;
        } else if (inexact) {
          const unsigned long long idx = atomicAdd(tp.exact_count, 1ull);
          tp.exact_rows[idx] = make_int2(static_cast<int>(row), nb);
          any = true;
        }
      }
      // fixed-order tile sum over the 4 first-half warps: one named barrier,
      // partial slots double-buffered by tile parity
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      const unsigned anyw = __ballot_sync(0xffffffffu, any);
      if (lane == 0) {
        red[tb * 4 + quad] = s;
        red_flag[tb * 4 + quad] = anyw != 0;
      }
      named_bar(2 + grp, 128);
      if (quad == 0 && lane == 0) {
        p.tile_sum[t] = ((red[tb * 4] + red[tb * 4 + 1]) + red[tb * 4 + 2]) + red[tb * 4 + 3];
        p.tile_flag[t] = red_flag[tb * 4] | red_flag[tb * 4 + 1] | red_flag[tb * 4 + 2] | red_flag[tb * 4 + 3];
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem_base);
}

// ---------------------------------------------------------------- prep --------
// B pieces: mu~ = mu * 2^-em split into fp16 hi + lo, [Kp][Dp] zero padded; column
// bias for the ranking (sqeuclid p_k, cosine 0, padding +inf).
__global__ void prep_b_kernel(const double* __restrict__ stats, int k, int d, int kp, int dp, bool cos,
                              float smu, __half* bh, __half* bl, float* colbias, float* munorm,
                              double4* clu) {
  const int c = blockIdx.x;
  const double n = c < k ? fmax(stats[c], 1.0) : 1.0;
  const double* sums = stats + (cos ? k : 2 * k) + static_cast<int64_t>(c) * d;
  for (int l = threadIdx.x; l < dp; l += blockDim.x) {
    float h = 0.f, lo = 0.f;
    if (c < k && l < d) {
      const double mu = sums[l] / n * static_cast<double>(smu);
      const __half hh = __double2half(mu);
      h = __half2float(hh);
      lo = static_cast<float>(mu - static_cast<double>(h));
    }
    bh[static_cast<int64_t>(c) * dp + l] = __float2half_rn(h);
    bl[static_cast<int64_t>(c) * dp + l] = __float2half_rn(lo);
  }
  __shared__ double red[4];
  double sq = 0.0;
  if (c < k)
    for (int l = threadIdx.x; l < d; l += blockDim.x) {
      const double mu = sums[l] / n;
      sq += mu * mu;
    }
  for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    colbias[c] = c < k ? (cos ? 0.0f : static_cast<float>(stats[k + c] / n)) : INFINITY;
    munorm[c] = __double2float_ru(sqrt(red[0] + red[1] + red[2] + red[3]) * (1.0 + 1e-12));
    if (c < k) clu[c] = make_double4(n, n > 1.0 ? 1.0 / (n - 1.0) : 0.0, cos ? 0.0 : stats[k + c], 0.0);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    FSIL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (!ptr || q != cudaDriverEntryPointSuccess) fail(FSIL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

CUtensorMap make_map_2d(CUtensorMapDataType dt, const void* ptr, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(FSIL_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

int pick_bn(int k) { return k <= 32 ? 32 : k <= 64 ? 64 : 128; }

size_t tc_smem(int bn, int kp) {
  const size_t ring = bn <= 32 ? TcCfg<32>::kRing : bn <= 64 ? TcCfg<64>::kRing : TcCfg<128>::kRing;
  return 1024 + ring + 26 * 8 + 2 * BM * 8 + 8 * BM * 4 + 128 + static_cast<size_t>(ncb_bn_pad(kp)) * 4;
}

template <int BN, bool COS>
void launch_tc(fsil_context* c, const CUtensorMap& mx, const CUtensorMap& mh, const CUtensorMap& ml,
               const TcParams& tp, int64_t ntiles) {
  auto kern = score_tc_kernel<BN, COS>;
  const size_t smem = tc_smem(BN, tp.ncb * BN);
  FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, c->num_sms));
  kern<<<grid, kThreads, smem, c->stream>>>(mx, mh, ml, tp, ntiles);
  FSIL_LAUNCHED(c);
}

}  // namespace

bool tc_supported(const fsil_context* c) {
  const int bn = pick_bn(c->k);
  const int kp = (c->k + bn - 1) / bn * bn;
  return c->d % 4 == 0 && c->n < (int64_t(1) << 31) && c->k >= 2 && tc_smem(bn, kp) <= c->smem_optin;
}

int64_t tc_tiles(const fsil_context* c, int* tile_rows) {
  *tile_rows = BM;
  return (c->n + BM - 1) / BM;
}

void score_tc(fsil_context* c, const ScoreParams& p) {
  const bool cos = c->metric == FSIL_COSINE;
  const int bn = pick_bn(c->k);
  const int ncb = (c->k + bn - 1) / bn;
  const int kp = ncb * bn;
  const int nkc = (c->d + BK - 1) / BK;
  const int dp = nkc * BK;
  // global power-of-two scalings: max|x~| and max|mu~| in [2^14, 2^15)
  float h_bound[4] = {0, 0, 0, 0}, h_xmax = 0.f;
  FSIL_CUDA(cudaMemcpyAsync(h_bound, c->bound.p, sizeof(h_bound), cudaMemcpyDeviceToHost, c->stream));
  FSIL_CUDA(cudaMemcpyAsync(&h_xmax, c->xmax.p, sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  FSIL_CUDA(cudaStreamSynchronize(c->stream));
  const int ex = h_xmax > 0.f ? std::ilogb(h_xmax) - 14 : 0;
  const int em = h_bound[2] > 0.f ? std::ilogb(h_bound[2]) - 14 : 0;
  c->tc_b.ensure(2ull * kp * dp * sizeof(__half) + 2ull * kp * sizeof(float) + kp * sizeof(double4) + 64);
  __half* bh = c->tc_b.as<__half>();
  __half* bl = bh + static_cast<size_t>(kp) * dp;
  float* colbias = reinterpret_cast<float*>(bl + static_cast<size_t>(kp) * dp);
  float* munorm = colbias + kp;
  double4* clu = reinterpret_cast<double4*>((reinterpret_cast<uintptr_t>(munorm + kp) + 31) & ~uintptr_t(31));
  prep_b_kernel<<<kp, 128, 0, c->stream>>>(p.stats, c->k, c->d, kp, dp, cos, std::ldexp(1.0f, -em), bh, bl,
                                           colbias, munorm, clu);
  FSIL_LAUNCHED(c);
  const CUtensorMap mx = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, c->X, c->d, c->n, c->d * 4ull, 32, BM);
  const CUtensorMap mh = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, bh, dp, kp, dp * 2ull, BK, bn);
  const CUtensorMap ml = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, bl, dp, kp, dp * 2ull, BK, bn);
  TcParams tp{};
  tp.p = p;
  tp.ncb = ncb;
  tp.nkc = nkc;
  tp.sx = std::ldexp(1.0f, -ex);
  tp.smul = std::ldexp(1.0f, ex + em);
  tp.smul64 = std::ldexp(1.0, ex + em);
  tp.colbias = colbias;
  tp.munorm = munorm;
  tp.clu = clu;
  // |dot error| <= cdot*||x||*||mu|| + floor: split residuals 3*2^-22 relative; fp32
  // accumulation of the main term over ceil(D/16) MMA steps at 2^-24 (the correction
  // accumulator holds values <= 2^-10 of it); the final main+correction add; and the
  // fp16 subnormal floor 2^-25 per element in scaled units (sqrt(D) via Cauchy-Schwarz).
  const float u = 5.9604645e-8f;
  const float steps = static_cast<float>((c->d + 15) / 16);
  tp.cdot = 1.05f * (12.0f + steps + 1.0f + 2.0f * steps / 512.0f) * u;
  tp.floor_coef = 1.05f * 0.5f * u * std::sqrt(static_cast<float>(c->d)) *
                  (std::ldexp(1.0f, em) + std::ldexp(1.0f, ex) * h_bound[0] / std::max(h_xmax, 1e-30f));
  tp.mu_max = h_bound[0];
  tp.p_max = h_bound[1];
  c->exact_rows.ensure(std::max<int64_t>(c->n, 1) * sizeof(int2));
  c->exact_count.ensure(sizeof(unsigned long long));
  FSIL_CUDA(cudaMemsetAsync(c->exact_count.p, 0, sizeof(unsigned long long), c->stream));
  tp.exact_rows = c->exact_rows.as<int2>();
  tp.exact_count = c->exact_count.as<unsigned long long>();
  const int64_t ntiles = (c->n + BM - 1) / BM;
  if (cos) {
    if (bn == 32) launch_tc<32, true>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 64) launch_tc<64, true>(c, mx, mh, ml, tp, ntiles);
    else launch_tc<128, true>(c, mx, mh, ml, tp, ntiles);
  } else {
    if (bn == 32) launch_tc<32, false>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 64) launch_tc<64, false>(c, mx, mh, ml, tp, ntiles);
    else launch_tc<128, false>(c, mx, mh, ml, tp, ntiles);
  }
  c->tc_exact_used = true;
}

}  // namespace fsil
