// score_tc.cuh -- definitions shared by the tcgen05 scoring kernels: the single-CTA
// kernel (score_tc.cu) and the CTA-pair kernel for large cluster tables (score_tc2.cu).
#pragma once

#include <cuda_fp16.h>

#include "score_common.cuh"
#include "sm100.cuh"

namespace fsil {
namespace tc {

using namespace sm100;


constexpr int BM = 128;               // rows per tile = TMEM lanes
constexpr int BK = 64;                // fp16 K elements per chunk (one 128-byte swizzle row)
constexpr int kStgBytes = 2 * BM * 128;  // two fp32 boxes of 32 columns
constexpr int kABytes = BM * 128;        // one fp16 A piece (hi or lo)
constexpr int kThreads = 640;            // 20 warps (5 warpgroups)

__host__ __device__ constexpr int ncb_bn_pad(int kp) { return (kp + 3) & ~3; }

// Operand scalings and error-bound constants, computed on the device by prep_b from
// the derived bounds (no host round trip between aggregation and scoring).
struct TcScale {
  double smul64;          // 2^(ex+em): dot = acc * smul
  float sx;               // 2^-ex: x -> x~
  float smul;
  float floor_mu;         // fp16 subnormal floor of the mu pieces, per unit ||x||
  float floor_x;          // fp16 subnormal floor of the x pieces, per unit ||mu|| (absolute in x)
  float mu_max;           // max ||mu_k||
  float p_max;            // max p_k (sqeuclid)
  int thr_g;              // threshold mode: the extra K step's power-of-two slot exponent g
};

struct TcParams {
  ScoreParams p;
  int ncb, nkc;           // cluster blocks, K chunks
  const float* colbias;   // [ncb*BN]: sqeuclid p_k, cosine 0, padding +inf
  const __half* munorm;   // [ncb*BN]: ||mu_k|| / mu_max rounded up (neighbour error bounds)
  int nstg;               // X staging stages
  int nsa;                // decoupled mode: A operand slots (0: A converted in place in the X stages)
  int dual;               // two MMA-issuing warps (alternate tiles; TS mode only)
  const TcScale* scale;
  float cdot;             // relative dot bound coefficient
  unsigned long long* dbg;  // optional per-role wait-cycle counters (FSIL_TC_PROFILE)
  int split;              // separate correction accumulator (large D)
  uint8_t* ascratch;      // streaming mode: [grid][nkc][kStgBytes] converted A chunks (or null)
  float exic;             // ||x||^2 relative error / u: 8.1 (fp32 blocks of 8), +2.1 on fp64 input
  const double* xi_rows;  // per-row fp64 ||x||^2 from the aggregation pass (or null: converters form it)
  long long* trace;       // FSIL_TRACE builds: per-tile role timestamps of CTA 0 (or null)
  int lean;               // converters only convert; the epilogue fetches own/||x||^2 itself
  int2* pair_rows;        // T3: rows whose neighbour is one of {nb, .y} (certified pair)
  unsigned long long* pair_count;
  const float* lmnorm;    // [ncb*BN] ||mu_k - hm_k|| (mu units, rounded up): one-MMA level bound
  const float* lmmax;     // max_k lmnorm
  // threshold mode (sqeuclid, D <= 48, several cluster blocks; score_tc.cu "threshold scan"):
  // one extra K step adds t_row + q_k to every accumulator, so the sign bit alone says
  // whether column k is within the row's certified threshold
  int thr;                // 0 off; else the first fp16 column of the extra K step (16 ceil(D/16))
  const uint4* thr_t;     // [n] per row: the 8 fp16 A slots of t_row (thr_kernel)
  int nbs;                // threshold mode: B operand stages (0: the block-size default)
  int astg;               // threshold mode: bytes per A stage (16 KB when only box 0 / the hi piece is staged; else 32 KB)
  int bres;               // threshold mode: the whole hi-piece table stays in shared memory (no B ring)
  int wshift;             // role ids rotated by this many warps (0 or a multiple of 4): logical warp = (physical + wshift) % 20
  int thr_l1;             // threshold mode: MMAs per K step -- 3 (fp16x3) or 1 (hx.hm only; the dropped pieces are in the row's margin)
  int4* cand_rows;        // [n] threshold mode: a row's second to fourth candidate columns (when nb[row]'s top bits say 2..4)
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// Neighbour certification of one row from the epilogue's running keys (the ranking key
// m' = m - rowc: sqeuclid m = xi + p_k - 2 dot, cosine m = 1 - dot/||x||; row constant
// dropped, no clamp).  b1 <= b2 (<= b3, T3) are the best keys, arg / arg2 their columns;
// mu_arg_ratio = ||mu_arg|| / max ||mu|| rounded up.  The key error bound per unit ||x||
// for a column of norm ||mu||: cdot ||mu|| (split residuals + truncating fp32
// accumulation, see score_tc) + floor_mu (mu pieces' fp16 subnormal floor) + floor_x
// ||mu|| / ||x|| (x pieces' floor, absolute in x: per row).  Writes the nominated
// neighbour; uncertain rows go to the fp64 refinement (flag_rows) or, T3, to the
// certified-pair list when every other column is clearly behind.
template <bool COS, bool T3>
__device__ __forceinline__ bool certify_row(const TcParams& tp, const TcScale& sc, int64_t row, int own,
                                            float xi, float xn, float rnf, float b1, float b2, float b3,
                                            int arg, int arg2, float mu_arg_ratio, float mu_arg2_ratio = 1.0f,
                                            float x_rel = -1.0f, float lm_arg = 0.0f, float lm_arg2 = 0.0f,
                                            float lm_any = 0.0f) {
  const float u = 5.9604645e-8f;
  const float rowc = COS ? 1.0f : xi;
  const float exi = tp.exic * u * xi;  // ||x||^2 error (fp32 blocks of 8; fp64 input rounding)
  const float rx = COS ? rnf : rsqrtf(xi);  // 1/||x|| (<= 2.2u; inf for a zero row -> flagged)
  // x_rel >= 0 (two-MMA first level): the dropped x piece's ||lx||/||x~||, which also covers
  // the x pieces' fp16 subnormal floor; otherwise that floor per row
  const float cmu = tp.cdot + (x_rel >= 0.0f ? x_rel : sc.floor_x * rx * 1.0001f);
  // key error: the dot bound (per unit ||x|| for cosine); the key's own roundings
  // (cosine: rsqrt 2.2u + product 0.5u + fma 0.5u on |m| <= 1, within 4u(|b1|+1));
  // the ||x||^2 error
  // one-MMA level (lm_* > 0): the dropped hx.lm piece, ||hx|| ||mu_k - hm_k||, ||hx|| <=
  // (1 + x_rel) ||x~||, per column (the winner, the runner-up) or its maximum (any column)
  const float lmf = 1.0f + fmaxf(x_rel, 0.0f);
  const float eps_dot1 = cmu * sc.mu_max + sc.floor_mu + lmf * lm_any;  // any column, per unit ||x||
  const float eps_m = COS ? (eps_dot1 + 4.0f * u * (fabsf(b1) + 1.0f) + tp.exic * u)
                          : (2.0f * eps_dot1 * xn + 3.0f * u * (fabsf(b1) + sc.p_max + 2.0f * xn * sc.mu_max) + exi);
  // the winner's key error uses its own cluster norm (the runner-up's column is
  // not tracked: any-column bound eps_m)
  const float mu_arg = mu_arg_ratio * sc.mu_max;
  const float eps_dot1_arg = cmu * mu_arg + sc.floor_mu + lmf * lm_arg;
  const float eps_m_arg = COS ? (eps_dot1_arg + 4.0f * u * (fabsf(b1) + 1.0f) + tp.exic * u)
                              : (2.0f * eps_dot1_arg * xn + 3.0f * u * (fabsf(b1) + sc.p_max + 2.0f * xn * sc.mu_max) + exi);
  // neighbour certain: clear gap, and no tie through the clamps at 0 (and 2).  With the
  // top-3 (T3) the runner-up's own norm bounds its key and every other column is at or
  // behind b3 with the any-column bound: certain when min(b2 - e2, b3 - e_any) > b1 + e_arg.
  bool gap_ok = (b2 - b1) > eps_m + eps_m_arg && rowc + b2 > eps_m;
  if (T3 && arg2 >= 0) {
    const float eps_dot1_2 = cmu * (mu_arg2_ratio * sc.mu_max) + sc.floor_mu + lmf * lm_arg2;
    const float eps_m_2 = COS ? (eps_dot1_2 + 4.0f * u * (fabsf(b1) + 1.0f) + tp.exic * u)
                              : (2.0f * eps_dot1_2 * xn + 3.0f * u * (fabsf(b1) + sc.p_max + 2.0f * xn * sc.mu_max) + exi);
    gap_ok = gap_ok || (fminf(b2 - eps_m_2, b3 - eps_m) > b1 + eps_m_arg && rowc + b2 > eps_m_2 && rowc + b3 > eps_m);
  }
  const bool full = !gap_ok || arg < 0 || (COS && !(rowc + b1 < 2.0f - eps_m));
  tp.p.nb[row] = arg >= 0 ? arg : (own == 0 ? 1 : 0);  // the refinement rewrites flagged rows
  // T3: the neighbour is one of the top two when every other column is clearly
  // behind the winner (third-best gap, no clamp tie) -- two fp64 means decide it
  const bool pair = T3 && full && arg >= 0 && arg2 >= 0 && (b3 - b1) > eps_m + eps_m_arg &&
                    (rowc + b3 > eps_m) && (!COS || rowc + b1 < 2.0f - eps_m);
  if (pair) {
    const unsigned long long idx = atomicAdd(tp.pair_count, 1ull);
    tp.pair_rows[idx] = make_int2(static_cast<int>(row), arg2);
  } else if (full) {
    const unsigned long long idx = atomicAdd(tp.p.flag_count, 1ull);
    tp.p.flag_rows[idx] = static_cast<int32_t>(row);
  }
  return !full;  // the nominated neighbour is certain
}

// Tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry point).
CUtensorMap make_map_2d(CUtensorMapDataType dt, const void* ptr, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B);

// The CTA-pair kernel (score_tc2.cu): M = 256 rows per pair, N = 256 cluster columns per
// MMA block, for streaming cluster tables.  Returns false when it does not apply.
bool pair_supported(const fsil_context* c, const TcParams& tp, int bn);
void launch_tc_pair(fsil_context* c, const CUtensorMap& mx, const CUtensorMap& mh, const CUtensorMap& ml,
                    TcParams tp, int64_t ntiles, bool cos, bool t3, int l1);

}  // namespace tc
}  // namespace fsil
