// score_common.cuh -- fp64 reference formulas shared by the scoring, refinement
// and tensor-core epilogues.  Operation order follows the reference exactly:
//   sqeuclid foreign: xi + Psi_k/n - (2*cross)/n, max(0, .)      squared_euclidean.cpp:79,81
//   sqeuclid own    : (n*xi + Psi - 2*cross)/(n - 1), max(0, .)   squared_euclidean.cpp:77,81
//   cosine foreign  : 1 - cross/n, clamp [0, 2]                   cosine.cpp:85,87
//   cosine own      : (n - cross)/(n - 1), clamp [0, 2]           cosine.cpp:83,87
// (cross = Y_k . x for sqeuclid, Omega_k . (x/||x||) for cosine.)
#pragma once

#include "device_util.cuh"
#include "fsil_internal.cuh"

namespace fsil {

struct ScoreParams {
  const float* X;         // fp32 features (the fast scoring pass)
  const double* X64;      // fp64 front end: the caller's exact features (null for fp32 input)
  const int32_t* dense;
  int64_t n;
  int d, dp, k;
  int xstride;            // floats per staged row in shared memory
  int nstage;             // x tile buffers per CTA (1 or 2)
  const float* mu32;      // [kpad][dp]
  const float* p32;       // [kpad]
  const double* stats;    // fp64 all-reduced stats (StatsLayout)
  const double* nk;       // [k]
  const float* bound;     // [0] max ||mu||, [1] max p
  double* s;              // required (internal buffer if the caller passes none)
  int32_t* nb;
  int32_t* own;
  double* a;
  double* b;
  double* tile_sum;       // [ntiles]
  int32_t* tile_flag;     // [ntiles]
  int32_t* flag_rows;     // [n]
  unsigned long long* flag_count;
  const int* abort;       // set on the device when this call's K speculation missed: the
                          // scoring kernels return at entry (their inputs are not a dataset's)
};

// Feature element idx (row * d + l) as the exact-path kernels see it: the caller's
// fp64 value on the fp64 front end, else the fp32 input widened.
__device__ __forceinline__ double xval(const ScoreParams& p, int64_t idx) {
  return p.X64 ? p.X64[idx] : static_cast<double>(p.X[idx]);
}

// fp32 bound constant gamma_m = m u / (1 - m u), u = 2^-24.
__device__ __forceinline__ float gamma_f32(int m) {
  const float mu = static_cast<float>(m) * 5.9604645e-8f;
  return mu / (1.0f - mu);
}

__device__ __forceinline__ double sq_foreign(double xi, double psi, double n, double cross) {
  return fmax(0.0, xi + psi / n - 2.0 * cross / n);
}
__device__ __forceinline__ double sq_own(double xi, double psi, double n, double cross) {
  return fmax(0.0, (n * xi + psi - 2.0 * cross) / (n - 1.0));
}
__device__ __forceinline__ double cos_foreign(double n, double cross) {
  return fmin(fmax(1.0 - cross / n, 0.0), 2.0);
}
__device__ __forceinline__ double cos_own(double n, double cross) {
  return fmin(fmax((n - cross) / (n - 1.0), 0.0), 2.0);
}

// Exact (fp64) a_i, b_i, s_i for a row given its own and neighbour cluster.
// x is read through a generic pointer (shared or global memory).
template <bool COS>
__device__ __forceinline__ void exact_row(const float* x, int d, int own, int nb,
                                          const double* stats, const double* nk, int k,
                                          double& a, double& b, double& s) {
  const double* sums = stats + (COS ? k : 2 * k);
  const double* yo = sums + static_cast<int64_t>(own) * d;
  const double* yb = sums + static_cast<int64_t>(nb) * d;
  double ss = 0.0, co = 0.0, cb = 0.0;
  for (int l = 0; l < d; ++l) {
    const double v = x[l];
    ss = fma(v, v, ss);
    co = fma(__ldg(yo + l), v, co);
    cb = fma(__ldg(yb + l), v, cb);
  }
  const double n_o = nk[own], n_b = nk[nb];
  const bool singleton = n_o == 1.0;
  if (COS) {
    const double nrm = sqrt(ss);
    b = cos_foreign(n_b, cb / nrm);
    a = singleton ? 0.0 : cos_own(n_o, co / nrm);
  } else {
    b = sq_foreign(ss, stats[k + nb], n_b, cb);
    a = singleton ? 0.0 : sq_own(ss, stats[k + own], n_o, co);
  }
  s = singleton ? 0.0 : assemble_score(a, b);
}

}  // namespace fsil
