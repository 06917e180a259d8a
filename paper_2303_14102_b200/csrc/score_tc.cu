// score_tc.cu -- K3: per-point scoring on the 5th-generation tensor cores.
//
// Replaces score_range + mean_dist_to_cluster + make_point_score
// (squared_euclidean.cpp:65-108, cosine.cpp:71-117, report.cpp:16-30) when
// X . mu^T is a real contraction.  One persistent CTA per SM, warp-specialised:
//
//   warp 0      TMA producer: fp32 X boxes (128 rows x 32 cols, 128B swizzle) into a
//               staging ring; fp16 cluster-mean pieces B_hi/B_lo into the operand ring
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer (kind::f16, fp32 accum)
//   warps 2..5  epilogue (one TMEM lane = one row): ranking keys, top-2 with a
//               certified error bound -> the nominated neighbour cluster
//   warps 6..9  converters: x (fp32) -> x*2^-ex split into fp16 hi + lo in the UMMA
//               K-major SWIZZLE_128B layout, plus ||x||^2 (fp32 and fp64) per row
//
// Split precision ("fp16x3"): x~ = hx + lx, mu~ = hm + lm (exact to ~2^-22 after a
// global power-of-two scaling); dot = hx.hm + hx.lm + lx.hm, three MMAs per K step.
// Every row carries a certified bound on its dots; rows whose neighbour is not
// certain go to the fp64 argmin refinement (K4).  This pass only NOMINATES the
// neighbour: a_i, b_i and s_i of every row come from the fp64 exact pass
// (finalize.cu), so no tensor-core rounding reaches s_i or S.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>

#include "score_tc.cuh"

namespace fsil {
namespace {

using namespace sm100;
using namespace tc;

// Timeline tracing (compile with -DFSIL_TRACE, run with FSIL_TC_TRACE=1): CTA 0 records
// clock64() at fixed points of each role for its first 64 tiles.
#ifdef FSIL_TRACE
#define TRACE(i, k)                                                                                  \
  do {                                                                                               \
    if (blockIdx.x == 0 && tp.trace && (threadIdx.x & 31) == 0 && (i) < 64) tp.trace[(i) * 9 + (k)] = clock64(); \
  } while (0)
#else
#define TRACE(i, k) \
  do {              \
  } while (0)
#endif

template <int BN>
struct TcCfg {
  static constexpr int kBStg = BN <= 32 ? 4 : BN <= 64 ? 3 : 2;  // B (hi+lo) operand stages
  static constexpr int kBBytes = BN * 128;
  static constexpr size_t kBRing = static_cast<size_t>(kBStg) * 2 * kBBytes;
};

// Optional wait profiling (FSIL_TC_PROFILE): cycles each role spends blocked, per
// barrier (slots 0..8), added straight to global counters so the normal build keeps
// no per-thread state for it.
#define TW(slot, bar, par)                                                          \
  do {                                                                              \
    if (PROF && dbgp) {                                                             \
      const long long t0__ = clock64();                                             \
      mbar_wait(bar, par);                                                          \
      if (lane == 0) atomicAdd(dbgp + (slot), static_cast<unsigned long long>(clock64() - t0__)); \
    } else {                                                                        \
      mbar_wait(bar, par);                                                          \
    }                                                                               \
  } while (0)

// Warp roles (warpgroup aligned, so each group can set its own register budget):
//   warpgroup 0: warp 0 X producer (TMA), warp 1 TMEM owner + MMA issuer, warp 2 B
//                producer (TMA), warp 3 idle -- 40 registers
//   warpgroups 1-2 (warps 4..11): epilogue, two groups of four -- 120 registers
//   warpgroups 3-4 (warps 12..19): converters -- 96 registers
constexpr int kEpiWarp0 = 4, kConvWarp0 = 12;

__device__ __forceinline__ bool elect_one_sync() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(pred));
  return pred != 0;
}
#ifndef FSIL_EPI_REGS
#define FSIL_EPI_REGS 136
#endif
#ifndef FSIL_CONV_REGS
#define FSIL_CONV_REGS 72
#endif
#ifndef FSIL_WG0_REGS
#define FSIL_WG0_REGS 64
#endif
// CTA register pool per lane: 4 x 40 + 8 x epilogue + 8 x converters <= 20 x 96
static_assert(4 * FSIL_WG0_REGS + 8 * FSIL_EPI_REGS + 8 * FSIL_CONV_REGS <= 20 * 96, "register split exceeds the pool");

// KC: columns of each 32-column chunk the epilogue scans (BN = 32 with K <= 24 skips
// the padding columns; otherwise 32)
// EG: epilogue groups.  3 only in decoupled mode at BN = 32 (C2): warps 4..15 are three
// groups of four taking tiles round-robin, warps 16..19 the converters (one row each).
// T3: the epilogue also tracks the third-best key and the runner-up's column, so a row
// whose top-2 is uncertain but whose third-best is clear resolves as a certified pair (two
// fp64 foreign means) instead of a full K x D refinement (large cluster tables, C5).
// THR: threshold mode (see "threshold mode" below): one extra K step per cluster block, the
// converters add the row's t slots, the epilogue only harvests sign bits.
template <int BN, bool COS, bool PROF, int KC, int EG = 2, bool T3 = false, bool THR = false>
__global__ void __launch_bounds__(kThreads, 1)
    score_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_bh,
                    const __grid_constant__ CUtensorMap tmap_bl, TcParams tp, int64_t ntiles) {
  griddep_wait();           // (PDL) prep_b's operands and every earlier phase are visible
  if (*tp.p.abort) return;  // K speculation missed: the call is repeated
  using C = TcCfg<BN>;
  // B operand stages: the block-size default, or (threshold mode) more of them -- there a
  // cluster block is a handful of MMAs, so the ring must cover the L2 latency of its refills
  // (one-MMA threshold level: only the hi piece is staged, so the same ring space holds
  // twice the stages at half the stride)
  const int bstr = (THR && tp.thr_l1 == 1) ? C::kBBytes : 2 * C::kBBytes;
  const int NB = THR && tp.nbs ? tp.nbs * (2 * C::kBBytes / bstr) : C::kBStg;
  const int nbring = THR && tp.nbs ? tp.nbs : C::kBStg;  // ring space in (hi + lo) stage units
  // X stages: a TMA-filled fp32 box pair that the converters overwrite in place with
  // the fp16 A pieces (hi over box 0, lo over box 1), freed by the MMA commit
  const int NS = tp.nstg;
  // Decoupled (NSA > 0; one cluster block, ||x||^2 from the aggregation pass): the
  // converters read a stage into registers and free it at once, then write the A
  // pieces into one of NSA separate operand slots that the MMA commit frees -- the X
  // stages only cover TMA latency instead of being held through conversion and MMA.
  const int NSA = tp.nsa;
  constexpr int kConv0 = kEpiWarp0 + 4 * EG;  // first converter warp
  constexpr int kConvWarps = 20 - kConv0;     // 8 (EG = 2) or 4 (EG = 3)
  // TS: the two epilogue groups take alternate tiles, each with its own pair of
  // accumulator buffers, so consecutive tiles' epilogues overlap -- for tiles of at
  // most two cluster blocks (with more, the MMA stream would serialise on one
  // group's buffers).  Otherwise the groups split the column chunks of every tile,
  // cycling through `nacc` buffers (4 when they fit the 512 TMEM columns).
  const uint32_t astride = tp.split ? 2 * BN : BN;  // TMEM columns per accumulator buffer
  // (threshold mode: always alternate tiles -- its issuer interleaves the cluster blocks of
  // two tiles, one per group, so neither group's buffer pair serialises the MMA stream)
  const bool TS = THR || (tp.ncb <= 2 && 4 * astride <= 512);
  const uint32_t nacc = 4 * astride <= 512 ? 4 : 2;
  // A-resident: a tile's converted A chunks stay in their stages for every cluster
  // block (X read and converted once per tile); otherwise re-staged per block
  const bool ares = tp.ncb > 1 && 2 * tp.nkc <= NS;
  const int xpasses = ares ? 1 : tp.ncb;
  // A-scratch (streaming, several cluster blocks): the first pass over a tile's K
  // chunks converts X and also bulk-stores each converted stage to this CTA's global
  // (L2-resident) scratch; the later passes bulk-load the converted chunks instead of
  // re-staging and re-converting X
  // (nkc >= NS: a slot is rewritten only after the MMA consumed its previous load)
  // (several cluster blocks per tile only occur at BN = 128: compiled out otherwise)
  uint8_t* const scr = (BN == 128 && !ares && tp.ncb > 1 && tp.nkc >= NS) ? tp.ascratch : nullptr;
  uint8_t* const myscr = scr ? scr + static_cast<size_t>(blockIdx.x) * tp.nkc * kStgBytes : nullptr;
  constexpr uint32_t kTmemCols = BN <= 32 ? 256 : 512;
  constexpr uint32_t kIdesc = idesc_f16_f32(BM, BN);
  const ScoreParams& p = tp.p;

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by a pointer offset (keeps the shared address space visible to
  // the compiler: LDS/STS rather than generic accesses)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // (threshold mode at D <= 32 with the hi piece only: a stage is one 16 KB box)
  const int stgb = THR ? tp.astg : kStgBytes;
  const bool bres = THR && tp.bres;  // the whole hi-piece table resident: [ncb][kBBytes], loaded once
  uint8_t* stg = base;                      // [NS][stgb]
  uint8_t* aslot = stg + NS * stgb;         // [NSA][kStgBytes] decoupled A operand slots
  uint8_t* bring = aslot + NSA * kStgBytes; // [NB][b_hi | b_lo]
  uint64_t* bars = reinterpret_cast<uint64_t*>(bring + (bres ? tp.ncb * C::kBBytes : nbring * 2 * C::kBBytes));
  uint64_t* stg_full = bars;               // [NS <= 8] X landed (TMA)
  uint64_t* stg_empty = bars + 8;          // [NS] stage free (MMA commit)
  uint64_t* a_full = bars + 16;            // [NS] A pieces written (converters) -- [NSA] decoupled
  uint64_t* a_empty = stg_empty + NS;      // decoupled: [NSA] A slot free (MMA commit); NS + NSA <= 8
  uint64_t* b_full = bars + 24;            // [NB]
  uint64_t* b_empty = bars + 28;           // [NB]
  uint64_t* acc_full = bars + 32;          // [6]
  uint64_t* acc_empty = bars + 38;         // [6]
  uint64_t* meta_full = bars + 44;         // [2]
  uint64_t* meta_empty = bars + 46;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 48);
  uint64_t* scr_ready = bars + 49;         // [1] a tile's converted chunks are in scratch
  double* meta_xi = reinterpret_cast<double*>(bars + 50);   // [2][2][BM] ||x||^2 halves
  float* part = reinterpret_cast<float*>(meta_xi + 4 * BM);  // [2][5][BM] second-half partial top-2/3
  int* meta_own = reinterpret_cast<int*>(part + 10 * BM);     // [2][BM] own cluster per row
  float* cb_s = reinterpret_cast<float*>(meta_own + 2 * BM);  // [ncb*BN] column bias
  __half* mn_s = reinterpret_cast<__half*>(cb_s + ncb_bn_pad(tp.ncb * BN));  // [ncb*BN] ||mu_k||/mu_max, rounded up

  // Role ids rotated by tp.wshift warps (a multiple of 4: the setmaxnreg warpgroups and the
  // epilogue's TMEM lane quadrants keep their alignment): an experiment switch that puts the
  // producers and MMA issuers (logical warps 0-3) on the physical warps 16-19.
  const int tid = tp.wshift ? static_cast<int>((threadIdx.x + 32u * tp.wshift) % kThreads) : static_cast<int>(threadIdx.x);
  const int warp = tid >> 5, lane = tid & 31;
  const int ncb = tp.ncb, nkc = tp.nkc;
  unsigned long long* const dbgp = PROF ? tp.dbg : nullptr;  // compiled out unless profiling
  const long long t_start = dbgp ? clock64() : 0;
  for (int j = tid; j < ncb * BN; j += blockDim.x) {
    cb_s[j] = tp.colbias[j];
    mn_s[j] = tp.munorm[j];
  }
  const TcScale sc = *tp.scale;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(stg_full + i, 1);
      mbar_init(stg_empty + i, NSA ? kConvWarps : 1);
      mbar_init(a_full + i, myscr ? 1 : kConvWarps);
    }
    for (int i = 0; i < NSA; ++i) mbar_init(a_empty + i, 1);
    for (int i = 0; i < NB; ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, THR ? 2 : 1);  // (threshold mode: both issuers release a stage)
    }
    for (int i = 0; i < 2 * EG; ++i) {
      mbar_init(acc_full + i, 1);
      mbar_init(acc_empty + i, TS ? 4 : 8);
    }
    mbar_init(scr_ready, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(meta_full + i, 8);
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

  if (warp < kEpiWarp0) {
    if (FSIL_WG0_REGS != 96) setmaxnreg_dec<FSIL_WG0_REGS>();
    if (warp == 0 && lane == 0) {
      // ---------------------------------------------------------- TMA producer: X
      uint32_t n1 = 0, ntl = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++ntl) {
        const int row0 = static_cast<int>(t * BM);
        for (int xp = 0; xp < xpasses; ++xp) {
          if (myscr && xp == 1) {  // first pass converted and stored: wait, then reuse
            TW(0, scr_ready, ntl & 1);
            fence_proxy_async_global();
          }
          for (int kc = 0; kc < nkc; ++kc, ++n1) {
            const int s1 = n1 % NS;
            const int nbox = (kc * BK + 32 < p.d) ? 2 : 1;
            TW(0, stg_empty + s1, ((n1 / NS) & 1) ^ 1);
            if (myscr && xp > 0) {
              mbar_arrive_expect_tx(a_full + s1, kStgBytes);
              bulk_load(stg + s1 * kStgBytes, myscr + static_cast<size_t>(kc) * kStgBytes, kStgBytes, a_full + s1);
              continue;  // (no stg_full phase: the converters count TMA'd items per stage)
            }
            mbar_arrive_expect_tx(stg_full + s1, nbox * BM * 128);
            for (int b = 0; b < nbox; ++b)
              tma_load_2d(stg + s1 * stgb + b * BM * 128, &tmap_x, stg_full + s1, kc * BK + b * 32, row0);
            TRACE(ntl, 0);
          }
        }
      }
    } else if (warp == 2 && lane == 0 && !(THR && EG == 3)) {
      // ---------------------------------------------------------- TMA producer: B pieces
      uint32_t n2 = 0;
      if (bres) {  // the table once: every block's hi piece, one barrier
        mbar_arrive_expect_tx(b_full, static_cast<uint32_t>(ncb) * C::kBBytes);
        for (int cb = 0; cb < ncb; ++cb) tma_load_2d(bring + cb * C::kBBytes, &tmap_bh, b_full, 0, cb * BN);
      }
      // (threshold mode: a B block serves two tiles, see the issuer)
      for (int64_t t = blockIdx.x; t < ntiles && !bres; t += (THR ? 2 : 1) * static_cast<int64_t>(gridDim.x)) {
        for (int cb = 0; cb < ncb; ++cb) {
          for (int kc = 0; kc < nkc; ++kc, ++n2) {
            const int sb = n2 % NB;
            uint8_t* bs = bring + sb * bstr;
            TW(1, b_empty + sb, ((n2 / NB) & 1) ^ 1);
            if (THR && tp.thr_l1 == 1) {  // one-MMA threshold level: the hi piece only
              mbar_arrive_expect_tx(b_full + sb, C::kBBytes);
              tma_load_2d(bs, &tmap_bh, b_full + sb, kc * BK, cb * BN);
              continue;
            }
            mbar_arrive_expect_tx(b_full + sb, 2 * C::kBBytes);
            tma_load_2d(bs, &tmap_bh, b_full + sb, kc * BK, cb * BN);
            tma_load_2d(bs + C::kBBytes, &tmap_bl, b_full + sb, kc * BK, cb * BN);
            TRACE((t - blockIdx.x) / gridDim.x, 8);
          }
        }
      }
    } else if (THR && (warp == 1 || warp == 3 || (EG == 3 && warp == 2))) {
      // ---------------------------------------------------------- MMA issuers, threshold mode:
      // one K chunk, A-resident tiles; a cluster block is D/16 + 1 (or 3 D/16 + 1) MMAs, so
      // the issue path itself must stay short -- incremental ring positions (no division),
      // operand descriptors by offset from one base per ring, and the whole warp runs the
      // loop (every value warp-uniform: descriptors stay in uniform registers) while one
      // elected lane issues.  Two tiles at a time: each B block is loaded once for both;
      // warp 1 issues tile 2i into epilogue group 0's buffer pair, warp 3 tile 2i + 1 into
      // group 1's, so the two issue streams (whose per-block waits are latency, not work)
      // overlap, and both groups scan concurrently with no merge between them.  A B stage is
      // free when both issuers' MMAs on it retired (b_empty counts two).
      // Three groups (EG = 3; only with the resident table, so warp 2 has no B ring to feed:
      // it loads the table once and issues for group 2): three tiles at a time, ONE
      // accumulator per group -- a group's MMAs and scan alternate, the three groups overlap.
      const int g = warp == 1 ? 0 : warp == 3 ? 1 : 2;
      if (EG == 3 && warp == 2) {
        if (lane == 0) {
          mbar_arrive_expect_tx(b_full, static_cast<uint32_t>(ncb) * C::kBBytes);
          for (int cb = 0; cb < ncb; ++cb) tma_load_2d(bring + cb * C::kBBytes, &tmap_bh, b_full, 0, cb * BN);
        }
        __syncwarp();
      }
      const int nks = (p.d + 15) >> 4;
      const uint64_t da0 = desc_k_sw128(smem_u32(stg)), db0 = desc_k_sw128(smem_u32(bring));
      const uint32_t xo = static_cast<uint32_t>(tp.thr) >> 3;  // the extra K step, in descriptor units (16 B)
      const int l1 = tp.thr_l1;
      int s1 = 0, sb = 0;
      uint32_t ph1 = 0, phb = 0, ngc = 0;
      auto adv_a = [&](int k) {
        s1 += k;
        while (s1 >= NS) {
          s1 -= NS;
          ph1 ^= 1u;
        }
      };
      if (g) adv_a(g);
      const int64_t nmine = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
      for (int64_t i = 0; i < nmine; i += EG) {
        const bool have = i + g < nmine;  // (the last pair may lack its second tile)
        const uint64_t dah = da0 + static_cast<uint32_t>(s1) * (static_cast<uint32_t>(stgb) >> 4), dal = dah + (kABytes >> 4);
        if (have) TW(5, a_full + s1, ph1);
        if (bres && i == 0) TW(3, b_full, 0u);  // the resident table has landed
        for (int cb = 0; cb < ncb; ++cb) {
          if (bres) {
            if (have) {
              const uint64_t dbh = db0 + static_cast<uint32_t>(cb) * (C::kBBytes >> 4);
              const int ab = EG == 3 ? g : 2 * g + static_cast<int>(ngc & 1u);
              TW(2, acc_empty + ab, (EG == 3 ? (ngc & 1u) : ((ngc >> 1) & 1u)) ^ 1u);
              ++ngc;
              tc_fence_after();
              const uint32_t dacc = tmem_base + ab * astride;
              if (elect_one_sync()) {
                if (nks == 2) {
                  mma_f16(dacc, dah, dbh, kIdesc, 0u);
                  mma_f16(dacc, dah + 2, dbh + 2, kIdesc, 1u);
                } else {
                  for (int ks = 0; ks < nks; ++ks) mma_f16(dacc, dah + 2 * ks, dbh + 2 * ks, kIdesc, ks > 0 ? 1u : 0u);
                }
                mma_f16(dacc, dah + xo, dbh + xo, kIdesc, 1u);  // + t_row + q_k
                mma_commit(acc_full + ab);
                if (cb == ncb - 1) mma_commit(stg_empty + s1);
              }
              __syncwarp();
            }
            continue;
          }
          TW(3, b_full + sb, phb);
          if (have) {
            const uint64_t dbh = db0 + static_cast<uint32_t>(sb) * (static_cast<uint32_t>(bstr) >> 4), dbl = dbh + (C::kBBytes >> 4);
            const int ab = 2 * g + static_cast<int>(ngc & 1u);
            TW(2, acc_empty + ab, ((ngc >> 1) & 1u) ^ 1u);
            ++ngc;
            tc_fence_after();
            const uint32_t dacc = tmem_base + ab * astride;
            if (elect_one_sync()) {
              if (l1 == 1) {  // hx.hm only
                if (nks == 2) {
                  mma_f16(dacc, dah, dbh, kIdesc, 0u);
                  mma_f16(dacc, dah + 2, dbh + 2, kIdesc, 1u);
                } else {
                  for (int ks = 0; ks < nks; ++ks) mma_f16(dacc, dah + 2 * ks, dbh + 2 * ks, kIdesc, ks > 0 ? 1u : 0u);
                }
              } else {
                for (int ks = 0; ks < nks; ++ks) {
                  mma_f16(dacc, dah + 2 * ks, dbh + 2 * ks, kIdesc, ks > 0 ? 1u : 0u);
                  mma_f16(dacc, dah + 2 * ks, dbl + 2 * ks, kIdesc, 1u);
                  mma_f16(dacc, dal + 2 * ks, dbh + 2 * ks, kIdesc, 1u);
                }
              }
              mma_f16(dacc, dah + xo, dbh + xo, kIdesc, 1u);  // + t_row + q_k
              mma_commit(acc_full + ab);
              mma_commit(b_empty + sb);
              if (cb == ncb - 1) mma_commit(stg_empty + s1);
            }
          } else if (elect_one_sync()) {
            mbar_arrive(b_empty + sb);  // nothing of this stage is read by this issuer
          }
          __syncwarp();
          if (++sb == NB) {
            sb = 0;
            phb ^= 1u;
          }
        }
        adv_a(EG);
      }
    } else if (warp == 1 && lane == 0 && !(TS && NSA)) {
      // ---------------------------------------------------------- MMA issuer (column-split
      // epilogue or in-place A stages: C3/C4/C5).  A/B-measured: this form is 3-5% faster
      // there than the ring-counter issuer below, which wins with decoupled A slots (C2).
      uint32_t n2 = 0, na = 0, ng0 = 0, ng1 = 0, nt = 0, nx = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
        for (int cb = 0; cb < ncb; ++cb, ++na) {
          int ab;
          uint32_t ph;
          if (TS) {
            const int g = nt & 1;
            const uint32_t cnt = g ? ng1 : ng0;  // per-group buffer-pair counters
            ab = 2 * g + (cnt & 1);
            ph = (cnt >> 1) & 1;
            ng0 += g ? 0u : 1u;
            ng1 += g ? 1u : 0u;
          } else {
            ab = na % nacc;
            ph = (na / nacc) & 1;
          }
          TW(2, acc_empty + ab, ph ^ 1);
          tc_fence_after();
          const uint32_t d_main = tmem_base + ab * astride, d_corr = tp.split ? d_main + BN : d_main;
          for (int kc = 0; kc < nkc; ++kc, ++n2) {
            const uint32_t ia = ares ? nx + kc : nx + cb * nkc + kc;  // A item
            const int s1 = static_cast<int>(ia % NS), sb = n2 % NB;
            if (!ares || cb == 0) TW(3, a_full + s1, (ia / NS) & 1);
            TW(3, b_full + sb, (n2 / NB) & 1);
            tc_fence_after();
            const int rem = p.d - kc * BK;
            const int nks = rem >= BK ? 4 : (rem + 15) / 16;
            const uint32_t ah = smem_u32(stg + s1 * kStgBytes), al = ah + kABytes;
            const uint32_t bh = smem_u32(bring + sb * 2 * C::kBBytes), bl = bh + C::kBBytes;
            for (int ks = 0; ks < nks; ++ks) {
              const uint32_t off = ks * 32;
              const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
              // split: the two correction terms (~2^-10 of the main term) accumulate
              // separately so their fp32 rounding is ~2^-10 smaller; for small D a
              // single accumulator is certified tightly enough and is cheaper
              mma_f16(d_main, desc_k_sw128(ah + off), desc_k_sw128(bh + off), kIdesc, acc0);
              mma_f16(d_corr, desc_k_sw128(ah + off), desc_k_sw128(bl + off), kIdesc, tp.split ? acc0 : 1u);
              mma_f16(d_corr, desc_k_sw128(al + off), desc_k_sw128(bh + off), kIdesc, 1u);
            }
            // threshold mode: the extra K step (hi pieces only) adds t_row + q_k
            if (THR && kc == nkc - 1)
              mma_f16(d_main, desc_k_sw128(ah + 2 * tp.thr), desc_k_sw128(bh + 2 * tp.thr), kIdesc, 1u);
            mma_commit(b_empty + sb);                               // B stage free when these retire
            if (!ares || cb == ncb - 1) mma_commit(stg_empty + s1);  // A stage: after its last use
          }
          mma_commit(acc_full + ab);  // accumulators ready for the epilogue
        }
        nx += ares ? nkc : ncb * nkc;
      }
    } else if ((warp == 1 || (warp == 3 && tp.dual)) && lane == 0 && TS && NSA) {
      // ---------------------------------------------------------- MMA issuer(s)
      // With alternating epilogue groups (TS) warps 1 and 3 issue the MMAs of even and
      // odd tiles respectively: each tile's operand slots, B stages and accumulator pair
      // are used by exactly one issuer, so the two streams need no ordering between them,
      // and the issue work (uniform-datapath descriptor arithmetic, waits) is halved per
      // issuing warp.  Both walk every tile to keep the ring counters in step.
      const uint32_t iid = warp == 3 ? 1u : 0u;
      const bool dual = TS && tp.dual;
      // ring positions (slot, phase) advance incrementally: no runtime division
      const int NA = NSA ? NSA : NS;
      uint8_t* const abuf = NSA ? aslot : stg;
      uint64_t* const a_free = NSA ? a_empty : stg_empty;
      int a_s = 0, b_s = 0;
      uint32_t a_ph = 0, b_ph = 0;
      auto adv = [](int& sl, uint32_t& ph, int n, int k) {
        sl += k;
        while (sl >= n) {
          sl -= n;
          ph ^= 1u;
        }
      };
      uint32_t na = 0, nt = 0, ngc[EG] = {};
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
        const bool mine = !dual || (nt & 1u) == iid;
        if (!mine) {  // the other issuer's tile: advance the counters only
          ngc[nt % EG] += ncb;
          na += ncb;
          adv(b_s, b_ph, NB, ncb * nkc);
          adv(a_s, a_ph, NA, ares ? nkc : ncb * nkc);
          continue;
        }
        int s_end = a_s;
        uint32_t ph_end = a_ph;
        for (int cb = 0; cb < ncb; ++cb, ++na) {
          int ab;
          uint32_t ph;
          if (TS) {
            const int g = static_cast<int>(nt % EG);
            const uint32_t cnt = ngc[g];  // per-group buffer-pair counters
            ab = 2 * g + (cnt & 1);
            ph = (cnt >> 1) & 1;
            ++ngc[g];
          } else {
            ab = na % nacc;
            ph = (na / nacc) & 1;
          }
          TW(2, acc_empty + ab, ph ^ 1);
          tc_fence_after();
          const uint32_t d_main = tmem_base + ab * astride, d_corr = tp.split ? d_main + BN : d_main;
          // A items of this block: the tile's chunks (A-resident: the same items for every
          // block), otherwise the next ncb*nkc items
          int sa = a_s;
          uint32_t pa = a_ph;
          if (!ares) adv(sa, pa, NA, cb * nkc);
          for (int kc = 0; kc < nkc; ++kc) {
            if (!ares || cb == 0) TW(3, a_full + sa, pa);
            TW(3, b_full + b_s, b_ph);
            TRACE(nt, 3);
            tc_fence_after();
            const int rem = p.d - kc * BK;
            // descriptors of the chunk's operand pieces; a 16-element K step is +32 B, i.e.
            // +2 in the descriptor's address field
            const uint64_t dah = desc_k_sw128(smem_u32(abuf + sa * kStgBytes)), dal = dah + (kABytes >> 4);
            const uint64_t dbh = desc_k_sw128(smem_u32(bring + b_s * 2 * C::kBBytes)), dbl = dbh + (C::kBBytes >> 4);
            const uint32_t acc_in = kc > 0 ? 1u : 0u;
            // split: the two correction terms (~2^-10 of the main term) accumulate
            // separately so their fp32 rounding is ~2^-10 smaller; for small D a
            // single accumulator is certified tightly enough and is cheaper
            if (rem >= BK) {
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
                const uint32_t acc0 = ks > 0 ? 1u : acc_in;
                mma_f16(d_main, dah + 2 * ks, dbh + 2 * ks, kIdesc, acc0);
                mma_f16(d_corr, dah + 2 * ks, dbl + 2 * ks, kIdesc, tp.split ? acc0 : 1u);
                mma_f16(d_corr, dal + 2 * ks, dbh + 2 * ks, kIdesc, 1u);
              }
            } else {
              const int nks = (rem + 15) / 16;
              for (int ks = 0; ks < nks; ++ks) {
                const uint32_t acc0 = ks > 0 ? 1u : acc_in;
                mma_f16(d_main, dah + 2 * ks, dbh + 2 * ks, kIdesc, acc0);
                mma_f16(d_corr, dah + 2 * ks, dbl + 2 * ks, kIdesc, tp.split ? acc0 : 1u);
                mma_f16(d_corr, dal + 2 * ks, dbh + 2 * ks, kIdesc, 1u);
              }
            }
            mma_commit(b_empty + b_s);                                 // B stage free when these retire
            if (!ares || cb == ncb - 1) mma_commit(a_free + sa);       // A stage / slot: after its last use
            adv(sa, pa, NA, 1);
            adv(b_s, b_ph, NB, 1);
          }
          s_end = sa;
          ph_end = pa;
          mma_commit(acc_full + ab);  // accumulators ready for the epilogue
          TRACE(nt, 4);
        }
        a_s = s_end;  // the tile's last A item + 1 (A-resident: the tile's nkc items)
        a_ph = ph_end;
      }
    }
  } else if (warp >= kConv0) {
    // (threshold mode with three groups: its converter loop is the two-group one, 80 registers,
    // and its scan needs fewer than the classic epilogue: 4 x 64 + 12 x 112 + 4 x 80 = the pool)
    constexpr int kConvRegs = EG == 3 ? (THR ? 80 : 56) : FSIL_CONV_REGS;
    static_assert(4 * FSIL_WG0_REGS + 12 * 120 + 4 * 56 <= 20 * 96, "EG = 3 register split exceeds the pool");
    static_assert(4 * FSIL_WG0_REGS + 12 * 112 + 4 * 80 <= 20 * 96, "threshold mode, EG = 3: register split exceeds the pool");
    if (kConvRegs != 96) setmaxnreg_dec<kConvRegs>();
    // ------------------------------------------------------------ converters (8 warps:
    // two threads per row; thread half hq reads fp32 box hq of the stage, then -- after
    // the whole group has read -- writes A chunks 4hq..4hq+3 of hi (over box 0) and lo
    // (over box 1))
    const int tl = tid - kConv0 * 32;
    const int r = tl & (BM - 1), hq = tl >> 7;  // row in tile, box / chunk half
    const int sw = r & 7;
    const float2 sx2 = make_float2(sc.sx, sc.sx), neg1 = make_float2(-1.f, -1.f);
    const bool unit_scale = sc.sx == 1.0f;  // prep_b picked no x scaling (EG = 3 path)
    uint32_t n1 = 0, nt = 0;
    int s1 = 0;        // n1 % NS, kept incrementally (NS is a runtime value)
    uint32_t ph1 = 0;  // (n1 / NS) & 1
    // ext: ||x||^2 comes from the aggregation pass and the epilogue fetches its per-row
    // inputs itself -- the converters only convert (no norm, no meta hand-off)
    const bool ext = tp.lean != 0;
    if (EG == 3 && !THR) {
      // decoupled, four converter warps (one thread per row, both 32-column boxes in
      // turn, two 16-byte units at a time -- 56 registers): wait for the stage and a free
      // A slot, convert, then free the stage and publish the slot
      const uint32_t wr = r * 128;
      int sa = 0;
      uint32_t pha = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < nkc; ++kc) {
          mbar_wait(stg_full + s1, ph1);
          mbar_wait(a_empty + sa, pha ^ 1);
          const uint8_t* sbase = stg + s1 * kStgBytes;
          uint8_t* abase = aslot + sa * kStgBytes;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            // box 1 of a last chunk with D - 64 kc <= 32 was not loaded, and the MMA's K
            // steps (nks) stop before it: its A pieces are neither written nor read
            if (h == 1 && kc * BK + 32 >= p.d) break;
            const uint8_t* srow = sbase + h * (BM * 128) + r * 128;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const float4 f0 = *reinterpret_cast<const float4*>(srow + (((2 * jj) ^ sw) << 4));
              const float4 f1 = *reinterpret_cast<const float4*>(srow + (((2 * jj + 1) ^ sw) << 4));
              const float v[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
              uint32_t hw[4], lw[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 x2 = make_float2(v[2 * e], v[2 * e + 1]);
                const float2 xx = unit_scale ? x2 : __fmul2_rn(x2, sx2);
                const __half2 hh = __float22half2_rn(xx);
                const float2 res = __ffma2_rn(__half22float2(hh), neg1, xx);  // exact
                const __half2 l = __float22half2_rn(res);
                hw[e] = *reinterpret_cast<const uint32_t*>(&hh);
                lw[e] = *reinterpret_cast<const uint32_t*>(&l);
              }
              const uint32_t pos = wr + (((4 * h + jj) ^ sw) << 4);
              *reinterpret_cast<uint4*>(abase + pos) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
              *reinterpret_cast<uint4*>(abase + BM * 128 + pos) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(stg_empty + s1);  // the stage has been read
            mbar_arrive(a_full + sa);
          }
          if (++s1 == NS) {
            s1 = 0;
            ph1 ^= 1;
          }
          if (++sa == NSA) {
            sa = 0;
            pha ^= 1;
          }
        }
      }
    } else if (NSA) {
      // decoupled: stage -> registers -> free the stage -> convert into an A slot
      const uint32_t rd = hq * (BM * 128) + r * 128, wr = r * 128;
      const bool tail_box = hq == 1;
      int sa = 0;
      uint32_t pha = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < nkc; ++kc) {
          mbar_wait(stg_full + s1, ph1);
          if (warp == kConv0) TRACE((t - blockIdx.x) / gridDim.x, 1);
          const uint8_t* sbase = stg + s1 * kStgBytes;
          float4 f[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) f[u] = *reinterpret_cast<const float4*>(sbase + rd + ((u ^ sw) << 4));
          __syncwarp();
          if (lane == 0) mbar_arrive(stg_empty + s1);  // the stage is in registers: TMA may refill it
          if (++s1 == NS) {
            s1 = 0;
            ph1 ^= 1;
          }
          if (tail_box && kc * BK + 32 >= p.d) {
#pragma unroll
            for (int u = 0; u < 8; ++u) f[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          mbar_wait(a_empty + sa, pha ^ 1);
          uint8_t* abase = aslot + sa * kStgBytes;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const float v[8] = {f[2 * jj].x,     f[2 * jj].y,     f[2 * jj].z,     f[2 * jj].w,
                                f[2 * jj + 1].x, f[2 * jj + 1].y, f[2 * jj + 1].z, f[2 * jj + 1].w};
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 xx = __fmul2_rn(make_float2(v[2 * e], v[2 * e + 1]), sx2);
              const __half2 h = __float22half2_rn(xx);
              const float2 res = __ffma2_rn(__half22float2(h), neg1, xx);  // exact
              const __half2 l = __float22half2_rn(res);
              hw[e] = *reinterpret_cast<const uint32_t*>(&h);
              lw[e] = *reinterpret_cast<const uint32_t*>(&l);
            }
            const uint32_t pos = wr + (((4 * hq + jj) ^ sw) << 4);
            *reinterpret_cast<uint4*>(abase + pos) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(abase + BM * 128 + pos) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(a_full + sa);
          if (warp == kConv0) TRACE((t - blockIdx.x) / gridDim.x, 2);
          if (++sa == NSA) {
            sa = 0;
            pha ^= 1;
          }
        }
      }
    } else if (THR) {
      // threshold mode (one K chunk, A-resident): the lean loop below, plus the extra K
      // step's A slots -- chunk jx = the row's t slots (thr_kernel), chunk jx + 1 = 2^g --
      // written by the thread whose half of the row holds those chunks
      const uint32_t rd = hq * (BM * 128) + r * 128, wr = r * 128;
      const bool tail_box = hq == 1;
      const int jx = tp.thr >> 3;
      // (three epilogue groups leave four converter warps: one thread per row, D <= 32, so the
      // row's second half holds nothing but the extra K step's slots -- written below)
      constexpr bool HALF = kConvWarps == 4;
      const bool mine = HALF || (jx >> 2) == hq;
      const uint32_t g1 = static_cast<uint32_t>(sc.thr_g + 15) << 10, g2 = g1 | (g1 << 16);  // fp16 2^g, twice
      const bool hi_only = tp.thr_l1 == 1;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t row = t * BM + r;
        const uint4 tsl = (mine && row < p.n) ? __ldg(tp.thr_t + row) : make_uint4(0u, 0u, 0u, 0u);
        TW(4, stg_full + s1, ph1);
        uint8_t* sbase = stg + s1 * stgb;
        float4 f[8];
        if (tail_box && 32 >= p.d) {  // box 1 absent (and, with 16 KB stages, not this stage's memory)
#pragma unroll
          for (int u = 0; u < 8; ++u) f[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) f[u] = *reinterpret_cast<const float4*>(sbase + rd + ((u ^ sw) << 4));
        }
        named_bar(5, HALF ? 128 : 256);  // every read of the stage precedes the in-place writes
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const float v[8] = {f[2 * jj].x,     f[2 * jj].y,     f[2 * jj].z,     f[2 * jj].w,
                              f[2 * jj + 1].x, f[2 * jj + 1].y, f[2 * jj + 1].z, f[2 * jj + 1].w};
          uint32_t hw[4], lw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 xx = __fmul2_rn(make_float2(v[2 * e], v[2 * e + 1]), sx2);
            const __half2 h = __float22half2_rn(xx);
            const float2 res = __ffma2_rn(__half22float2(h), neg1, xx);  // exact
            const __half2 l = __float22half2_rn(res);
            hw[e] = *reinterpret_cast<const uint32_t*>(&h);
            lw[e] = *reinterpret_cast<const uint32_t*>(&l);
          }
          const uint32_t pos = wr + (((4 * hq + jj) ^ sw) << 4);
          uint4 hv = make_uint4(hw[0], hw[1], hw[2], hw[3]);
          if (mine && 4 * hq + jj == jx) hv = tsl;
          if (mine && 4 * hq + jj == jx + 1) hv = make_uint4(g2, g2, g2, g2);
          *reinterpret_cast<uint4*>(sbase + pos) = hv;
          if (!hi_only) *reinterpret_cast<uint4*>(sbase + BM * 128 + pos) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        if (HALF && jx >= 4) {  // D = 32: the slots are chunks 4 and 5 of the row
          *reinterpret_cast<uint4*>(sbase + wr + ((jx ^ sw) << 4)) = tsl;
          *reinterpret_cast<uint4*>(sbase + wr + (((jx + 1) ^ sw) << 4)) = make_uint4(g2, g2, g2, g2);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full + s1);
        if (++s1 == NS) {
          s1 = 0;
          ph1 ^= 1;
        }
      }
    } else if (ext && !myscr && xpasses == 1) {
      // lean loop (every stage converted exactly once, nothing else): the per-thread
      // swizzled offsets are loop invariant
      const uint32_t rd = hq * (BM * 128) + r * 128, wr = r * 128;
      const bool tail_box = hq == 1;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kc = 0; kc < nkc; ++kc) {
          mbar_wait(stg_full + s1, ph1);
          uint8_t* sbase = stg + s1 * kStgBytes;
          float4 f[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) f[u] = *reinterpret_cast<const float4*>(sbase + rd + ((u ^ sw) << 4));
          if (tail_box && kc * BK + 32 >= p.d) {
#pragma unroll
            for (int u = 0; u < 8; ++u) f[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          named_bar(5, 256);  // every read of the stage precedes the in-place writes
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const float v[8] = {f[2 * jj].x,     f[2 * jj].y,     f[2 * jj].z,     f[2 * jj].w,
                                f[2 * jj + 1].x, f[2 * jj + 1].y, f[2 * jj + 1].z, f[2 * jj + 1].w};
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 xx = __fmul2_rn(make_float2(v[2 * e], v[2 * e + 1]), sx2);
              const __half2 h = __float22half2_rn(xx);
              const float2 res = __ffma2_rn(__half22float2(h), neg1, xx);  // exact
              const __half2 l = __float22half2_rn(res);
              hw[e] = *reinterpret_cast<const uint32_t*>(&h);
              lw[e] = *reinterpret_cast<const uint32_t*>(&l);
            }
            const uint32_t pos = wr + (((4 * hq + jj) ^ sw) << 4);
            *reinterpret_cast<uint4*>(sbase + pos) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(sbase + BM * 128 + pos) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(a_full + s1);
          if (++s1 == NS) {
            s1 = 0;
            ph1 ^= 1;
          }
        }
      }
    } else {
    // stg_full completes one phase per TMA'd item of a stage.  With the A scratch the
    // reloaded items in between never touch it, and they are issued at MMA pace, so a
    // parity derived from the running item count can alias two phases (the converters
    // run ahead of the barrier): the parity is tracked per stage over TMA'd items only.
    // Every TMA'd item of a stage is observed here, and the producer cannot land the next
    // one before this one was converted (scr_ready / stg_empty), so the waits never lag
    // the barrier by more than one phase.
    uint32_t tpar = 0;  // bit s: parity of stage s's next TMA'd item
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
      double xi = 0.0;
      // the epilogue's per-row inputs, fetched here off its critical path
      const int64_t row = t * BM + r;
      const int own = (hq == 0 && row < p.n) ? __ldg(p.dense + row) : -1;
      for (int xp = 0; xp < xpasses; ++xp) {
        if (myscr && xp > 0) {  // later passes load the stored conversions (producer)
          n1 += nkc;
          s1 = static_cast<int>(n1 % NS);
          continue;
        }
        for (int kc = 0; kc < nkc; ++kc, ++n1) {
          TW(4, stg_full + s1, (tpar >> s1) & 1u);
          tpar ^= 1u << s1;
          uint8_t* sbase = stg + s1 * kStgBytes;
          // (box 1 of the last chunk may be absent: those lanes read stale bytes, then zero
          // them on a warp-uniform branch rather than zero-initialising every chunk)
          float4 f[8];
          const uint8_t* srow = sbase + hq * (BM * 128) + r * 128;
#pragma unroll
          for (int u = 0; u < 8; ++u) f[u] = *reinterpret_cast<const float4*>(srow + ((u ^ sw) << 4));
          if (hq == 1 && kc * BK + 32 >= p.d) {
#pragma unroll
            for (int u = 0; u < 8; ++u) f[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          named_bar(5, 256);  // every read of the stage precedes the in-place writes
          uint8_t* hrow = sbase + r * 128;
          uint8_t* lrow = hrow + BM * 128;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {  // A chunk j = 8 fp16 = fp32 units 2jj, 2jj+1
            const int j = 4 * hq + jj;
            const float v[8] = {f[2 * jj].x,     f[2 * jj].y,     f[2 * jj].z,     f[2 * jj].w,
                                f[2 * jj + 1].x, f[2 * jj + 1].y, f[2 * jj + 1].z, f[2 * jj + 1].w};
            if (xp == 0 && !tp.xi_rows) {  // ||x||^2: fp32 blocks of 8 (error <= 8u each), fp64 across blocks
              float2 bs = make_float2(0.f, 0.f);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 ve = make_float2(v[2 * e], v[2 * e + 1]);
                bs = __ffma2_rn(ve, ve, bs);
              }
              xi += static_cast<double>(bs.x + bs.y);
            }
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // packed f32x2: scale (exact), hi, residual, lo
              const float2 xx = __fmul2_rn(make_float2(v[2 * e], v[2 * e + 1]), sx2);
              const __half2 h = __float22half2_rn(xx);
              const float2 res = __ffma2_rn(__half22float2(h), neg1, xx);  // exact
              const __half2 l = __float22half2_rn(res);
              hw[e] = *reinterpret_cast<const uint32_t*>(&h);
              lw[e] = *reinterpret_cast<const uint32_t*>(&l);
            }
            const int pos = (j ^ sw) << 4;
            *reinterpret_cast<uint4*>(hrow + pos) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(lrow + pos) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
          fence_proxy_async_smem();
          if (myscr) {
            // one thread: the converted stage -> scratch (source read before the MMA
            // may release the stage), then the single a_full arrival
            named_bar(5, 256);
            if (tl == 0) {
              bulk_store(myscr + static_cast<size_t>(kc) * kStgBytes, sbase, kStgBytes);
              bulk_wait_read();
              mbar_arrive(a_full + s1);
            }
          } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(a_full + s1);
          }
          if (++s1 == NS) {
            s1 = 0;
            ph1 ^= 1;
          }
        }
        if (myscr && tl == 0) {  // this tile's chunks are all in global memory
          bulk_wait_all();
          mbar_arrive(scr_ready);
        }
        if (xp == 0) {  // ||x||^2 halves and the own cluster to the epilogue
          const int tb = nt & 1;
          TW(6, meta_empty + tb, ((nt >> 1) & 1) ^ 1);
          meta_xi[(tb * 2 + hq) * BM + r] = xi;
          if (hq == 0) meta_own[tb * BM + r] = own;
          __syncwarp();
          if (lane == 0) mbar_arrive(meta_full + tb);
        }
      }
    }
    }
  } else {
    // ------------------------------------------------------------ epilogue (8 warps)
    setmaxnreg_inc<EG == 3 ? (THR ? 112 : 120) : FSIL_EPI_REGS>();  // CTA pool: see the static_asserts
    const int quad = warp & 3;                // TMEM lane quadrant of this warp
    const int r = quad * 32 + lane;           // row in tile
    const int grp = (warp - kEpiWarp0) >> 2;  // epilogue group 0 / 1
    uint32_t na = 0, nt = 0, ng = 0;
    constexpr int NQ = BN / 32;
    if (THR) {
      // ---- threshold mode: acc'' = x~.mu~_k + t_row + q_k; a clear sign bit = column k is
      // within the row's certified threshold.  Sign bits of a 32-column chunk are packed by
      // funnel shifts (four independent chains), then only the set bits are walked.
      const int64_t tstep = (TS ? EG : 1) * static_cast<int64_t>(gridDim.x);
      auto fetch_own = [&](int64_t tt) {
        const int64_t rr = tt * BM + r;
        return (tt < ntiles && rr < p.n) ? __ldg(p.dense + rr) : -1;
      };
      int own_n = fetch_own(blockIdx.x + (TS ? grp : 0) * static_cast<int64_t>(gridDim.x));
      // per row: four (hit mask, chunk base) slots in shared memory, [grp][slot][row] (two groups:
      // the meta_xi / part regions, unused in this mode); written and read by the row's own thread
      constexpr uint32_t kHitStride = BM * 8;
      static_assert(EG == 3 || 2 * 4 * kHitStride <= (4 * BM * 8 + 10 * BM * 4), "hit slots exceed the reused regions");
      // (three groups: 12 KB after the column norms, see tc_smem)
      const uint32_t hsb = EG == 3 ? ((smem_u32(mn_s + tp.ncb * BN) + 15u) & ~15u) : smem_u32(meta_xi);
      const uint32_t hs0 = hsb + static_cast<uint32_t>(grp) * 4u * kHitStride + static_cast<uint32_t>(r) * 8u;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
        const int tb = nt & 1;
        if (TS && static_cast<int>(nt % EG) != grp) continue;  // another group takes this tile
        const int64_t row = t * BM + r;
        const bool valid = row < p.n;
        const int own = own_n;
        own_n = fetch_own(t + tstep);
        // per row: up to four (chunk base, hit mask) slots, filled without branches; the
        // masks are decoded into columns once per tile
        uint32_t sp = 0;  // byte offset of the row's next (hit mask, chunk base) slot
        // the own column's chunk base and its cleared bit (own = -1: no chunk matches)
        const int okb = own & ~31;
        const uint32_t onot = ~(1u << (8 * (own & 3) + ((own & 31) >> 2)));
        auto harvest = [&](const uint32_t(&v)[32], int k0) {
          // sign bytes by byte permutes in sign-replication mode (0xff where the accumulator
          // is negative), four elements per word; word i contributes bit i of each byte:
          // bit 8c + i of `neg` <-> element 4i + c.  No shifts, no dependent chain longer
          // than the four-deep OR.
          uint32_t n0 = 0, n1 = 0;
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const uint32_t w0 = prmt(prmt(v[4 * i], v[4 * i + 1], 0xfbfbu), prmt(v[4 * i + 2], v[4 * i + 3], 0xfbfbu), 0x5410u);
            const uint32_t w1 = prmt(prmt(v[4 * i + 4], v[4 * i + 5], 0xfbfbu), prmt(v[4 * i + 6], v[4 * i + 7], 0xfbfbu), 0x5410u);
            n0 |= w0 & (0x01010101u << i);
            n1 |= w1 & (0x01010101u << (i + 1));
          }
          uint32_t hits = ~(n0 | n1);
          if (k0 == okb) hits &= onot;  // the own column never counts
          // a chunk with hits (rare) is appended to the row's shared-memory slots by a
          // predicated store: no branch, no vote, nothing else on the common path
          const bool hit = hits != 0u;
          if (hit && sp < 4u * kHitStride) st_shared_v2(hs0 + sp, hits, static_cast<uint32_t>(k0));
          sp += hit ? kHitStride : 0u;
        };
        uint32_t v[32], w[32];
        int pend_k0 = -1;  // chunk (in w) whose scan is still owed: the previous block's last
        for (int cb = 0; cb < ncb; ++cb) {
          int ab;
          uint32_t ph;
          if (TS && EG == 3) {  // (three groups: one accumulator each)
            ab = grp;
            ph = ng & 1;
            ++ng;
          } else if (TS) {
            ab = 2 * grp + (ng & 1);
            ph = (ng >> 1) & 1;
            ++ng;
          } else {  // (BN = 128, one accumulator per block: four buffers)
            ab = na & 3;
            ph = (na >> 2) & 1;
            ++na;
          }
          TW(8, acc_full + ab, ph);
          const long long ts0 = dbgp ? clock64() : 0;
          tc_fence_after();
          // The block's four 32-column chunks, software-pipelined: chunk q + 1 is in flight
          // while chunk q is scanned (tcgen05.wait::ld waits for every outstanding load, so
          // the overlap is load-vs-scan, one chunk deep), the previous block's last chunk is
          // scanned under this block's first load, and the accumulator goes back to the
          // issuer as soon as its last chunk is in registers.
          static_assert(!THR || BN == 128, "threshold scan: 128-column blocks");
          const uint32_t tb0 = tmem_base + ab * astride + (static_cast<uint32_t>(quad * 32) << 16);
          const int kb0 = cb * BN;
          tmem_ld32_issue(tb0, v);
          if (pend_k0 >= 0) harvest(w, pend_k0);
          tmem_ld_wait(v);
          tmem_ld32_issue(tb0 + 32, w);
          harvest(v, kb0);
          tmem_ld_wait(w);
          tmem_ld32_issue(tb0 + 64, v);
          harvest(w, kb0 + 32);
          tmem_ld_wait(v);
          tmem_ld32_issue(tb0 + 96, w);
          harvest(v, kb0 + 64);
          tmem_ld_wait(w);
          pend_k0 = kb0 + 96;
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty + ab);
          if (dbgp && warp == kEpiWarp0 && lane == 0) atomicAdd(dbgp + 12, static_cast<unsigned long long>(clock64() - ts0));
        }
        if (pend_k0 >= 0) harvest(w, pend_k0);
        // decode: columns of the set bits in ascending order (slots are in scan order), the
        // padding columns >= K dropped; more than four chunks with hits -> "more than four"
        int cnt = 0, c1 = -1, c2 = -1, c3 = -1, c4 = -1;
        {
          auto decode = [&](uint32_t hm, int kb) {
            while (hm) {
              const int j = __clz(hm);
              hm &= ~(0x80000000u >> j);
              const int col = kb + j;
              if (col < p.k) {
                c4 = cnt == 3 ? col : c4;
                c3 = cnt == 2 ? col : c3;
                c2 = cnt == 1 ? col : c2;
                c1 = cnt == 0 ? col : c1;
                ++cnt;
              }
            }
          };
          const uint32_t nh = sp / kHitStride;
          for (uint32_t i = 0; i < (nh < 4u ? nh : 4u); ++i) {
            uint32_t hm, kb;
            ld_shared_v2(hs0 + i * kHitStride, hm, kb);
            uint32_t nat = 0;  // back to scan order: bit 31 - e <-> element e
            while (hm) {
              const int b = __ffs(hm) - 1;
              hm &= hm - 1;
              nat |= 0x80000000u >> (4 * (b & 7) + (b >> 3));
            }
            decode(nat, static_cast<int>(kb));
          }
          if (nh > 4u) cnt = 5;
        }
        if (!TS) {  // merge the two column halves (group 1 -> smem -> group 0)
          int* pt = reinterpret_cast<int*>(part + tb * 5 * BM);  // double-buffered by tile parity
          if (grp == 1) {
            pt[0 * BM + r] = cnt;
            pt[1 * BM + r] = c1;
            pt[2 * BM + r] = c2;
            pt[3 * BM + r] = c3;
            pt[4 * BM + r] = c4;
          }
          named_bar(1, 256);
          if (grp == 1) continue;
          const int ocnt = pt[0 * BM + r];
          const int os[4] = {pt[1 * BM + r], pt[2 * BM + r], pt[3 * BM + r], pt[4 * BM + r]};
#pragma unroll
          for (int i = 0; i < 4; ++i) {  // the other half's hits follow this half's
            const int pos = cnt + i;
            c1 = pos == 0 ? os[i] : c1;
            c2 = pos == 1 ? os[i] : c2;
            c3 = pos == 2 ? os[i] : c3;
            c4 = pos == 3 ? os[i] : c4;
          }
          cnt += ocnt;
        }
        if (valid) {
          // the reference's neighbour is among the hits.  One -> certain.  Two to four ->
          // their columns go to cand_rows[row] and the count into the top bits of nb[row];
          // none (a row outside the slot range) or more -> code 1.  thr_resolve_kernel
          // (finalize.cu) scans nb afterwards: fp64 means of the candidates, or the fp64
          // refinement over all K for code 1 -- no atomics on this path.
          const int code = cnt == 1 ? 0 : (cnt >= 2 && cnt <= 4) ? cnt : 1;
          p.nb[row] = (cnt >= 1 ? c1 : (own == 0 ? 1 : 0)) | (code << 28);
          if (code >= 2) tp.cand_rows[row] = make_int4(c2, c3, c4, 0);
        }
      }
    } else {
    // Per-row inputs (own cluster; ||x||^2 when the aggregation pass provides it) are
    // fetched from global memory one tile ahead of their use, so their DRAM latency
    // overlaps the current tile instead of serialising with it.
    const int64_t tstep = (TS ? EG : 1) * static_cast<int64_t>(gridDim.x);
    int own_n = -1;
    double xi_n = 0.0;
    auto fetch = [&](int64_t tt) {
      const int64_t rr = tt * BM + r;
      const bool ok = tt < ntiles && rr < p.n;
      own_n = ok ? __ldg(p.dense + rr) : -1;
      xi_n = ok && tp.xi_rows ? __ldg(tp.xi_rows + rr) : 0.0;
    };
    if (tp.lean) fetch(blockIdx.x + (TS ? grp : 0) * static_cast<int64_t>(gridDim.x));
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
      const int tb = nt & 1;
      if (TS && static_cast<int>(nt % EG) != grp) continue;  // another group takes this tile
      const int64_t row = t * BM + r;
      const bool valid = row < p.n;
      int own;
      double xi64;
      // ||x||^2 from the aggregation pass (exact fp64) when it wrote one, issued early
      const double xi_g = (!tp.lean && tp.xi_rows && valid) ? __ldg(tp.xi_rows + row) : 0.0;
      if (tp.lean) {  // the lean converters hand nothing over: prefetched inputs
        own = own_n;
        xi64 = xi_n;
        fetch(t + tstep);
      } else {  // the converters' hand-off through shared memory
        TW(7, meta_full + tb, (nt >> 1) & 1);
        own = meta_own[tb * BM + r];
        xi64 = tp.xi_rows ? xi_g : meta_xi[(tb * 2) * BM + r] + meta_xi[(tb * 2 + 1) * BM + r];
      }
      const float xi = static_cast<float>(xi64);
      const float xn = COS ? 0.0f : sqrtf(xi);
      const float rnf = COS ? rsqrtf(xi) : 0.0f;  // 1/||x|| (MUFU.RSQ, <= 2.2u) for cosine
      // ranking key m' = m - rowc (row constant dropped, no clamp): sqeuclid
      // m = xi + p_k - 2 dot, cosine m = 1 - dot/||x||; dot = acc * smul
      const float rowm = COS ? -(sc.smul * rnf) : -2.0f * sc.smul;
      float b1 = INFINITY, b2 = INFINITY, b3 = INFINITY;
      int arg = -1, arg2 = -1;
      for (int cb = 0; cb < ncb; ++cb) {
        int ab;
        uint32_t ph;
        if (TS) {
          ab = 2 * grp + (ng & 1);
          ph = (ng >> 1) & 1;
          ++ng;
        } else {
          ab = na % nacc;
          ph = (na / nacc) & 1;
          ++na;
        }
        TW(8, acc_full + ab, ph);
        if (quad == 0) TRACE(nt, 5);
        const long long ts0 = dbgp ? clock64() : 0;
        tc_fence_after();
        // one 32-column chunk: ranking keys (own column excluded), running top-2
        auto scan32 = [&](const uint32_t(&v)[32], int k0) {
          const int ownrel = own - k0;
          int argc = -1;  // chunk-local index of a new best
          const float4* cb4 = reinterpret_cast<const float4*>(cb_s + k0);
#pragma unroll
          for (int j4 = 0; j4 < KC / 4; ++j4) {
            const float4 bias = cb4[j4];
            const float bj[4] = {bias.x, bias.y, bias.z, bias.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = 4 * j4 + e;
              const float acc = __uint_as_float(v[j]);
              float m = fmaf(acc, rowm, bj[e]);
              m = j == ownrel ? INFINITY : m;
              const bool lt = m < b1;  // strict: the lowest index keeps ties
              if (T3) {
                const bool lt2 = m < b2;
                arg2 = lt ? arg : (lt2 ? k0 + j : arg2);
                arg = lt ? k0 + j : arg;
                b3 = fminf(b3, fmaxf(b2, m));
              } else {
                argc = lt ? j : argc;
              }
              b2 = fminf(b2, fmaxf(b1, m));
              b1 = fminf(b1, m);
            }
          }
          if (!T3 && argc >= 0) arg = k0 + argc;
        };
        const int q0 = TS ? 0 : grp, qs = TS ? 1 : 2;
        const uint32_t tb0 = tmem_base + ab * astride + (static_cast<uint32_t>(quad * 32) << 16);
        if (tp.split) {
#pragma unroll 1
          for (int q = q0; q < NQ; q += qs) {
            uint32_t v[32], w[32];
            tmem_ld32_issue(tb0 + q * 32, v);
            tmem_ld32_issue(tb0 + q * 32 + BN, w);
            tmem_ld_wait2(v, w);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w[j]));
            scan32(v, cb * BN + q * 32);
          }
        } else {
#pragma unroll 1
          for (int q = q0; q < NQ; q += 2 * qs) {  // two chunks per TMEM wait
            uint32_t v[32], w[32];
            const bool two = q + qs < NQ;
            tmem_ld32_issue(tb0 + q * 32, v);
            if (two) tmem_ld32_issue(tb0 + (q + qs) * 32, w);
            tmem_ld_wait2(v, w);
            scan32(v, cb * BN + q * 32);
            if (two) scan32(w, cb * BN + (q + qs) * 32);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + ab);
        if (quad == 0) TRACE(nt, 6);
        if (dbgp && warp == kEpiWarp0 && lane == 0) atomicAdd(dbgp + 12, static_cast<unsigned long long>(clock64() - ts0));
      }
      const long long tf0 = dbgp ? clock64() : 0;
      if (!TS) {
        // ---- merge the two column halves (group 1 -> smem -> group 0)
        float* pt = part + tb * 5 * BM;  // double-buffered by tile parity
        if (grp == 1) {
          pt[0 * BM + r] = b1;
          pt[1 * BM + r] = b2;
          pt[2 * BM + r] = __int_as_float(arg);
          if (T3) {
            pt[3 * BM + r] = b3;
            pt[4 * BM + r] = __int_as_float(arg2);
          }
        }
        named_bar(1, 256);
        if (grp == 1) {
          __syncwarp();
          if (lane == 0 && !tp.lean) mbar_arrive(meta_empty + tb);
          continue;
        }
        const float c1 = pt[0 * BM + r], c2 = pt[1 * BM + r];
        const int a2 = __float_as_int(pt[2 * BM + r]);
        if (T3) {
          // merge the other half's (c1, a2), (c2, a2b), c3 into (b1, arg), (b2, arg2), b3:
          // lexicographic (key, column) order, so equal keys keep the lowest column
          const float c3 = pt[3 * BM + r];
          const int a2b = __float_as_int(pt[4 * BM + r]);
          auto before = [](float x, int ix, float y, int iy) { return x < y || (x == y && ix >= 0 && (iy < 0 || ix < iy)); };
          auto insert = [&](float m, int im) {
            b3 = fminf(b3, fmaxf(b2, m));
            if (before(m, im, b1, arg)) {
              b2 = b1;
              arg2 = arg;
              b1 = m;
              arg = im;
            } else if (before(m, im, b2, arg2)) {
              b2 = m;
              arg2 = im;
            }
          };
          insert(c1, a2);
          insert(c2, a2b);
          b3 = fminf(b3, c3);
        } else {
          const float nb1 = fminf(b1, c1);
          b2 = fminf(fminf(fmaxf(b1, c1), b2), c2);
          arg = (c1 < b1 || (c1 == b1 && a2 >= 0 && (arg < 0 || a2 < arg))) ? a2 : arg;
          b1 = nb1;
        }
      }
      __syncwarp();
      if (lane == 0 && !tp.lean) mbar_arrive(meta_empty + tb);

      // ---- neighbour certification.  The key error bound per unit ||x|| for a column of
      // norm ||mu||: cdot ||mu|| (split residuals + truncating fp32 accumulation, see
      // score_tc) + floor_mu (mu pieces' fp16 subnormal floor) + floor_x ||mu|| / ||x||
      // (x pieces' floor, absolute in x: per row, so rows far smaller than the shard's
      // largest element are still covered).  Uncertain rows go to the fp64 refinement.
      if (valid)
        certify_row<COS, T3>(tp, sc, row, own, xi, xn, rnf, b1, b2, b3, arg, arg2,
                             arg >= 0 ? __half2float(mn_s[arg]) : 1.0f,
                             (T3 && arg2 >= 0) ? __half2float(mn_s[arg2]) : 1.0f);
      if (dbgp && warp == kEpiWarp0 && lane == 0) atomicAdd(dbgp + 13, static_cast<unsigned long long>(clock64() - tf0));
      if (quad == 0 && lane == 0) TRACE(nt, 7);
    }
    }  // !THR
  }

  if (dbgp && lane == 0) {
    if (warp == 0) atomicAdd(dbgp + 9, static_cast<unsigned long long>(clock64() - t_start));
    if (warp == kEpiWarp0) atomicAdd(dbgp + 10, static_cast<unsigned long long>(clock64() - t_start));
    if (warp == kConv0) atomicAdd(dbgp + 11, static_cast<unsigned long long>(clock64() - t_start));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem_base);
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

}  // namespace

namespace tc {
CUtensorMap make_map_2d(CUtensorMapDataType dt, const void* ptr, uint64_t inner, uint64_t outer,
                        uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(FSIL_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}
}  // namespace tc

namespace {

// ---------------------------------------------------------------- prep --------
// Global power-of-two scalings chosen so max|x~| and max|mu~| lie in [2^14, 2^15):
// ex from max|x| of the shard, em from max|mu_kl| (derive's bound[2]).
__device__ __forceinline__ int scale_exp(float m, int target = 14) { return m > 0.f ? ilogbf(m) - target : 0; }

// fp16 slots of the threshold mode's extra K step: a value v (accumulator units) is carried
// as 6 equal high slots + a middle + a low slot, each times 2^g from the other operand:
// v ~ (6 h + m + l) 2^g, residuals exact in fp64, the low slot rounded up (so the carried
// value is >= v up to the slot's subnormal quantum).  |v| <= 6 * 65504 * 2^g or *ok = false.
__device__ __forceinline__ void thr_slots(double v, int g, __half (&out)[8], bool* ok) {
  const double s = ldexp(1.0, g);
  const double h0 = v / (6.0 * s);
  *ok = fabs(h0) <= 65504.0;
  const __half h = __double2half(h0);
  const double r1 = v - 6.0 * s * static_cast<double>(__half2float(h));
  const __half m = __double2half(r1 / s);
  const double r2 = r1 - s * static_cast<double>(__half2float(m));
  const __half l = __float2half_ru(__double2float_ru(r2 / s));
#pragma unroll
  for (int i = 0; i < 6; ++i) out[i] = h;
  out[6] = m;
  out[7] = l;
}

// B pieces: mu~ = mu * 2^-em split into fp16 hi + lo, [Kp][Dp] zero padded; column
// bias for the ranking (sqeuclid p_k, cosine 0, padding +inf); per-cluster norms (the
// winner's error bound); block 0 also writes the TcScale record the scoring kernel reads.
__global__ void prep_b_kernel(const double* __restrict__ stats, const float* __restrict__ bound,
                              const float* __restrict__ xmax, int k, int d, int kp, int dp, bool cos,
                              __half* bh, __half* bl, float* colbias, __half* munorm,
                              TcScale* scale, const int* abort, bool unit_ok, float* lmnorm, float* lmmax,
                              int thr_dx) {
  griddep_wait();
  if (*abort) return;
  const int c = blockIdx.x;
  // threshold mode: operands scaled to [2^12, 2^13) so dots (<= D 2^26) and the extra K
  // step's t and q slots stay within the fp16 slot range; em is raised further when p_max
  // alone would push |q| = p/2^(ex+em+1) past 2^32 (the mu pieces' floor term grows with it)
  const int tgt = thr_dx ? 12 : 14;
  int em = scale_exp(bound[2], tgt);
  const float xm = *xmax;
  // x needs no scaling when max|x| lies in [0.5, 2^14): x~ = x stays below fp16's max
  // and the subnormal floor of the small elements is in the per-row bound (floor_x);
  // the multiply-free converters then skip the multiply
  const int ex = (unit_ok && xm >= 0.5f && xm < 16384.f) ? 0 : scale_exp(xm, tgt);
  int thr_g = 0;
  if (thr_dx) {
    const float pm = bound[1];
    if (pm > 0.f) em = max(em, ilogbf(pm) + 1 - 33 - ex);
    const float qmax = ldexpf(pm, -(ex + em + 1));
    const float rmax = fmaxf(qmax, ldexpf(static_cast<float>(d), 26));
    thr_g = min(15, max(0, ilogbf(rmax) + 2 - 18));
  }
  const float smu = ldexpf(1.0f, -em);
  if (c == 0 && threadIdx.x == 0) {
    TcScale t;
    t.thr_g = thr_g;
    t.sx = ldexpf(1.0f, -ex);
    t.smul = ldexpf(1.0f, ex + em);
    t.smul64 = ldexp(1.0, ex + em);
    // fp16 subnormal floor: 2^-25 per element in scaled units, sqrt(D) via Cauchy-Schwarz:
    // |dot error| <= floor_mu ||x|| (mu pieces) + floor_x ||mu|| (x pieces)
    const float fl = 1.05f * 0.5f * 5.9604645e-8f * sqrtf(static_cast<float>(d));
    t.floor_mu = fl * ldexpf(1.0f, em);
    t.floor_x = fl * ldexpf(1.0f, ex);
    t.mu_max = bound[0];
    t.p_max = bound[1];
    *scale = t;
  }
  const double n = c < k ? fmax(stats[c], 1.0) : 1.0;
  const double* sums = stats + (cos ? k : 2 * k) + static_cast<int64_t>(c) * d;
  double lm2 = 0.0;  // ||mu~ - hm||^2: what a hm-only product leaves out (scaled units)
  for (int l = threadIdx.x; l < dp; l += blockDim.x) {
    float h = 0.f, lo = 0.f;
    if (c < k && l < d) {
      const double mu = sums[l] / n * static_cast<double>(smu);
      const __half hh = __double2half(mu);
      h = __half2float(hh);
      lo = static_cast<float>(mu - static_cast<double>(h));
      const double rem = mu - static_cast<double>(h);
      lm2 = fma(rem, rem, lm2);
    }
    if (thr_dx && l >= thr_dx && l < thr_dx + 16) {
      // extra K step (hi piece only): columns dx..dx+7 meet the row's t slots -> 2^g;
      // columns dx+8..dx+15 carry q_k = -p_k / 2^(ex+em+1) against the A side's 2^g
      // (padding clusters: the most negative value, never within a threshold)
      const int i = l - thr_dx;
      if (i < 8) {
        h = ldexpf(1.0f, thr_g);
      } else if (c < k) {
        __half qs[8];
        bool ok;
        thr_slots(-(stats[k + c] / n) * ldexp(1.0, -(ex + em + 1)), thr_g, qs, &ok);
        h = __half2float(qs[i - 8]);
      } else {
        h = -65504.0f;
      }
    }
    bh[static_cast<int64_t>(c) * dp + l] = __float2half_rn(h);
    bl[static_cast<int64_t>(c) * dp + l] = __float2half_rn(lo);
  }
  __shared__ double red[4];
  __shared__ double red2[4];
  for (int off = 16; off > 0; off >>= 1) lm2 += __shfl_xor_sync(0xffffffffu, lm2, off);
  if ((threadIdx.x & 31) == 0) red2[threadIdx.x >> 5] = lm2;
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
    const double nrm = sqrt(red[0] + red[1] + red[2] + red[3]) * (1.0 + 1e-12);
    // bound[0] = max ||mu_k|| rounded up, so the ratio is <= 1; every rounding upward
    munorm[c] = __float2half_ru(__double2float_ru(__ddiv_ru(nrm, fmax(static_cast<double>(bound[0]), 1e-300))));
    // ||mu - hm|| in mu units, rounded up (0 for padding columns)
    const double lmn = sqrt(red2[0] + red2[1] + red2[2] + red2[3]) * (1.0 + 1e-9) / static_cast<double>(smu);
    const float lmf = c < k ? __double2float_ru(lmn) : 0.0f;
    lmnorm[c] = lmf;
    atomicMax(reinterpret_cast<int*>(lmmax), __float_as_int(lmf));  // non-negative floats order as ints
  }
}

// ---------------------------------------------------------------- threshold mode ----
// (sqeuclid, D <= 48, several cluster blocks: C4.)  The scan's per-element work -- key,
// own-column exclusion, running top-2, argmin: 1 FFMA + 7 ALU operations -- paces the
// single-CTA kernel there (ncu: ALU pipe 77 %, tensor pipe 15 %).  Threshold mode moves the
// comparison into the tensor core.  Per row, thr_kernel evaluates in fp64 the ranking key
// m'_k = p_k - 2 x.mu_k of a few clusters near the row's own (nn_list_kernel: the centroid's
// nearest centroids); their minimum T is an upper bound of the row's true minimum over
// k != own.  One extra K step adds t_row = (T + margin) / 2^(ex+em+1) and q_k = -p_k /
// 2^(ex+em+1) to the accumulator x~.mu~_k, so
//     acc'' >= 0   <=>   m'_k (as the tensor core sees it) <= T + margin,
// and with `margin` = the certified error of that comparison every column that can be the
// reference's neighbour has a clear sign bit.  The epilogue packs the 32 sign bits of a chunk
// with one funnel shift per element and only walks the set bits: one hit -> that column is
// the neighbour, certain; two -> a certified pair (two fp64 means decide, pair_kernel); none
// or more -> the fp64 refinement over all K.  a_i, b_i, s_i come from the exact pass as
// always.  Which clusters enter T only affects how many rows have a single hit.
#ifndef FSIL_THR_M
#define FSIL_THR_M 16
#endif
constexpr int kThrM = FSIL_THR_M;  // candidate clusters per row
constexpr int kPieceRowsTc = 2048;  // = aggregate.cu's kPieceRows (rows per label-sorted piece)

// One block per cluster c: the kThrM clusters k != c with the smallest p_k - 2 mu_c.mu_k
// (fp32: a heuristic choice, no bound depends on it); fewer than kThrM others: repeated.
__global__ void __launch_bounds__(256) nn_list_kernel(const float* __restrict__ mu32, const float* __restrict__ p32,
                                                      int k, int d, int dp, int32_t* __restrict__ nn,
                                                      const int* abort) {
  griddep_wait();
  if (*abort) return;
  extern __shared__ float nsm[];  // [dp] mu_c, [k] keys
  float* muc = nsm;
  float* key = nsm + dp;
  __shared__ float rk[8];
  __shared__ int ri[8];
  const int c = blockIdx.x;
  for (int l = threadIdx.x; l < dp; l += blockDim.x) muc[l] = mu32[static_cast<int64_t>(c) * dp + l];
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const float* mj = mu32 + static_cast<int64_t>(j) * dp;
    float dot = 0.f;
    for (int l = 0; l < d; ++l) dot = fmaf(muc[l], mj[l], dot);
    key[j] = j == c ? INFINITY : p32[j] - 2.0f * dot;
  }
  __syncthreads();
  int last = c == 0 ? 1 : 0;
  for (int r = 0; r < kThrM; ++r) {
    float bk = INFINITY;
    int bi = -1;
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
      const float v = key[j];
      if (v < bk) {
        bk = v;
        bi = j;
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const float ok = __shfl_xor_sync(0xffffffffu, bk, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (oi >= 0 && (bi < 0 || ok < bk || (ok == bk && oi < bi))) {
        bk = ok;
        bi = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      rk[threadIdx.x >> 5] = bk;
      ri[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < 8; ++w)
        if (ri[w] >= 0 && (bi < 0 || rk[w] < bk || (rk[w] == bk && ri[w] < bi))) {
          bk = rk[w];
          bi = ri[w];
        }
      if (bi < 0) bi = last;  // fewer than kThrM other clusters (or non-finite keys): repeat
      last = bi;
      nn[c * kThrM + r] = bi;
      key[bi] = INFINITY;
    }
    __syncthreads();
  }
}

// Per row: T = min over the own cluster's candidate list of the key p_k - 2 x.mu_k (fp32, its
// rounding bounded below), the certified margin of the tensor-core comparison, and the 8 fp16
// A slots of t_row.  One block per piece of the label-sorted rows (<= 2048 rows of one
// cluster; a persistent grid strides the pieces): the candidates' means sit in shared memory
// (broadcast reads), one row per thread.
template <int D>
__global__ void __launch_bounds__(256, 4) thr_kernel(const float* __restrict__ X, const int32_t* __restrict__ rows,
                                                  int k, const int64_t* __restrict__ seg_begin,
                                                  const int64_t* __restrict__ seg_end,
                                                  const int64_t* __restrict__ piece_start, int piece_rows,
                                                  const float* __restrict__ mu32, const float* __restrict__ p32,
                                                  int dp, const int32_t* __restrict__ nn,
                                                  const TcScale* __restrict__ scale, float cdot,
                                                  const float* __restrict__ lmmax, uint4* __restrict__ thr_t,
                                                  const int* abort) {
  griddep_wait();
  if (*abort) return;
  __shared__ __align__(16) float cm[kThrM][D];  // candidate means (fp32 roundings)
  __shared__ float cp[kThrM];                   // ... and their p_k
  const int64_t total = piece_start[k];
  const TcScale sc = *scale;
  const double u = 5.9604645e-8;
  const double inv2s = 1.0 / (2.0 * sc.smul64);
  const double quantum = ldexp(1.0, sc.thr_g - 23) / inv2s;  // the slots' subnormal quantum, key units
  // one-MMA level (lmmax given): max_k ||mu_k - hm_k|| in mu units
  const double lm_any = lmmax ? static_cast<double>(*lmmax) * (1.0 + 1e-6) : -1.0;
  const float2 sx2 = make_float2(sc.sx, sc.sx), neg1 = make_float2(-1.f, -1.f);
  for (int64_t p = blockIdx.x; p < total; p += gridDim.x) {
    int lo = 0, hi = k - 1;  // cluster owning piece p: largest c with piece_start[c] <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (piece_start[mid] <= p) lo = mid;
      else hi = mid - 1;
    }
    const int c = lo;
    const int64_t b0 = seg_begin[c] + (p - piece_start[c]) * piece_rows;
    const int64_t b1 = min(seg_end[c], b0 + piece_rows);
    __syncthreads();  // the previous piece's reads of cm / cp are done
    for (int e = threadIdx.x; e < kThrM * D; e += blockDim.x) {
      const int j = e / D, l = e - j * D;
      cm[j][l] = mu32[static_cast<int64_t>(nn[c * kThrM + j]) * dp + l];
    }
    if (threadIdx.x < kThrM) cp[threadIdx.x] = p32[nn[c * kThrM + threadIdx.x]];
    __syncthreads();
    for (int64_t pos = b0 + threadIdx.x; pos < b1; pos += blockDim.x) {
      const int64_t r = rows[pos];
      const float4* xr = reinterpret_cast<const float4*>(X + r * D);
      float2 x[D / 2];
      float2 ss2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < D / 4; ++q) {
        const float4 f = ldg_stream(xr + q);
        x[2 * q] = make_float2(f.x, f.y);
        x[2 * q + 1] = make_float2(f.z, f.w);
        ss2 = __ffma2_rn(x[2 * q], x[2 * q], ss2);
        ss2 = __ffma2_rn(x[2 * q + 1], x[2 * q + 1], ss2);
      }
      // one-MMA level: ||lx||^2, lx = x~ - fp16(x~) (exact in fp32), in scaled units
      float2 ll2 = make_float2(0.f, 0.f);
      if (lm_any >= 0.0) {
#pragma unroll
        for (int q = 0; q < D / 2; ++q) {
          const float2 xx = __fmul2_rn(x[q], sx2);
          const float2 res = __ffma2_rn(__half22float2(__float22half2_rn(xx)), neg1, xx);
          ll2 = __ffma2_rn(res, res, ll2);
        }
      }
      float T = INFINITY;
#pragma unroll 4
      for (int j = 0; j < kThrM; ++j) {
        float2 a = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < D / 4; ++q) {
          const float4 m = *reinterpret_cast<const float4*>(&cm[j][4 * q]);
          a = __ffma2_rn(x[2 * q], make_float2(m.x, m.y), a);
          a = __ffma2_rn(x[2 * q + 1], make_float2(m.z, m.w), a);
        }
        T = fminf(T, fmaf(-2.0f, a.x + a.y, cp[j]));
      }
      const double ss = static_cast<double>(ss2.x + ss2.y);
      const double xn = sqrt(ss) * (1.0 + (D + 4) * u);  // >= ||x||
      // columns whose mean distance clamps to 0 tie with a clamped minimum: keep every
      // key <= -||x||^2 within the threshold too (squared_euclidean.cpp:81)
      const double Tm = fmax(static_cast<double>(T), -ss * (1.0 - (D + 4) * u));
      // T's own rounding: fp32 means (u each), the D-term fp32 dot (gamma_D), p_k (u), the
      // final fma (u) -- (2D + 5) u ||x|| max||mu|| + 3u max p.  The comparison: the three-MMA
      // dot bound (score_tc's cdot, the pieces' subnormal floors); the extra K step -- one
      // more MMA over |acc| + |t| + |q| (10.5u), the t and q slots' representation (2^-31
      // relative, their subnormal quantum) -- 24u of the magnitudes
      const double xm = xn * static_cast<double>(sc.mu_max);
      const double mag = fabs(Tm) + static_cast<double>(sc.p_max) + 2.0 * xm;
      const double edot = static_cast<double>(cdot) * xm + static_cast<double>(sc.floor_x) * sc.mu_max +
                          static_cast<double>(sc.floor_mu) * xn;
      const double e_t = (2.0 * D + 5.0) * u * xm + 3.0 * u * static_cast<double>(sc.p_max);
      // one-MMA level: x~.mu~ - hx.hm = hx.Lm + lx.mu~ with mu~ = hm + Lm, so per column
      // |dropped| <= (||x|| + ||lx||) ||Lm_k|| + ||lx|| ||mu_k|| (x and mu units)
      double e_drop = 0.0;
      if (lm_any >= 0.0) {
        const double lxn = sqrt(static_cast<double>(ll2.x + ll2.y)) * (1.0 + (D + 4) * u) / static_cast<double>(sc.sx);
        e_drop = (xn + lxn) * lm_any + lxn * static_cast<double>(sc.mu_max);
      }
      const double margin = 1.01 * (2.0 * (edot + e_drop) + e_t + 24.0 * u * mag + 4.0 * quantum);
      __half sl[8];
      bool ok;
      thr_slots((Tm + margin) * inv2s, sc.thr_g, sl, &ok);
      if (!ok || !(ss < INFINITY)) {
        // outside the slot range (or a non-finite row): no column can hit, so the row
        // goes to the fp64 refinement
#pragma unroll
        for (int i = 0; i < 8; ++i) sl[i] = __float2half_rn(-65504.0f);
      }
      uint4 o;
      o.x = static_cast<uint32_t>(__half_as_ushort(sl[0])) | (static_cast<uint32_t>(__half_as_ushort(sl[1])) << 16);
      o.y = static_cast<uint32_t>(__half_as_ushort(sl[2])) | (static_cast<uint32_t>(__half_as_ushort(sl[3])) << 16);
      o.z = static_cast<uint32_t>(__half_as_ushort(sl[4])) | (static_cast<uint32_t>(__half_as_ushort(sl[5])) << 16);
      o.w = static_cast<uint32_t>(__half_as_ushort(sl[6])) | (static_cast<uint32_t>(__half_as_ushort(sl[7])) << 16);
      thr_t[r] = o;
    }
  }
}

int pick_bn(int k) { return k <= 32 ? 32 : k <= 64 ? 64 : 128; }

// Shared memory with `nstg` X staging stages: operand ring, staging ring, barriers,
// meta_xi, merge partials, own clusters, column bias (fp32) and norms (fp16).
size_t tc_smem(int bn, int kp, int nstg, int nbs = 0, int astg = kStgBytes, size_t bres_bytes = 0, size_t extra = 0) {
  size_t bring = bn <= 32 ? TcCfg<32>::kBRing : bn <= 64 ? TcCfg<64>::kBRing : TcCfg<128>::kBRing;
  if (nbs) bring = static_cast<size_t>(nbs) * 2 * bn * 128;
  if (bres_bytes) bring = bres_bytes;
  return 1024 + bring + static_cast<size_t>(nstg) * astg + 50 * 8 + 4 * BM * 8 + 10 * BM * 4 + 2 * BM * 4 +
         static_cast<size_t>(ncb_bn_pad(kp)) * 4 + static_cast<size_t>(kp) * 2 + 16 + extra;
}
constexpr int kMaxStg = 8;
constexpr size_t kHitSlots3 = 3 * 4 * BM * 8 + 16;  // threshold mode, three groups: the rows' hit slots
int tc_stages(int bn, int kp, size_t optin) {
  int ns = kMaxStg;
  while (ns > 2 && tc_smem(bn, kp, ns) > optin) --ns;
  return ns;
}

// First-level MMAs per K step of the pair pass: FSIL_TC_L1 = 1 (default: hx.hm), 2 (hx.hm +
// hx.lm) or 3 (one three-MMA pass, no second level; FSIL_TC_TWO=0 is the same); fp64 inputs 3
static int pair_l1(const fsil_context* c) {
  static const int l1_env = [] {
    const char* e = std::getenv("FSIL_TC_L1");
    const char* t = std::getenv("FSIL_TC_TWO");
    if (t && std::atoi(t) == 0) return 3;
    return e ? std::max(1, std::min(3, std::atoi(e))) : 1;
  }();
  return c->X64 ? 3 : l1_env;
}

template <int BN, bool COS, int KC = 32, int EG = 2, bool T3 = false, bool THR = false>
void launch_tc(fsil_context* c, const CUtensorMap& mx, const CUtensorMap& mh, const CUtensorMap& ml,
               const TcParams& tp, int64_t ntiles, bool rec = true) {
  auto kern = tp.dbg ? score_tc_kernel<BN, COS, true, KC, EG, T3, THR> : score_tc_kernel<BN, COS, false, KC, EG, T3, THR>;
  const size_t smem = THR ? tc_smem(BN, tp.ncb * BN, tp.nstg, tp.nbs, tp.astg, tp.bres ? static_cast<size_t>(tp.ncb) * BN * 128 : 0,
                                  EG == 3 ? kHitSlots3 : 0)
                          : tc_smem(BN, tp.ncb * BN, tp.nstg + tp.nsa);
  if (c->timing && rec) {  // the kernel alone, for the roofline (ms_score_kernel)
    FSIL_CUDA(cudaEventRecord(c->ev[7], c->stream));
    c->ev7_recorded = true;
  }
  FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, c->num_sms));
  launch_pdl(c, kern, grid, kThreads, smem, mx, mh, ml, tp, ntiles);
}

// ---------------------------------------------------------------- two-level certificate
// Level 1 (the two-MMA CTA-pair pass) leaves its uncertain rows -- more than two candidate
// neighbours within its bound -- in flag_rows.  Level 2 gathers them into a compact matrix
// and re-scores them with this file's three-MMA kernel (split accumulators: the tight
// bound); its neighbours go back to the original rows, its certified pairs join the pair
// list, and only its own uncertain rows stay for the fp64 refinement.
__global__ void gather_uncertain_kernel(const float* __restrict__ X, const int32_t* __restrict__ dense,
                                        const int32_t* __restrict__ rows, int64_t nrows, int d,
                                        float* __restrict__ xs, int32_t* __restrict__ ds,
                                        unsigned long long* __restrict__ sub_counts) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x < 2) sub_counts[threadIdx.x] = 0ull;
  for (int64_t i = w; i < nrows; i += nw) {
    const int64_t r = rows[i];
    const float4* src = reinterpret_cast<const float4*>(X + r * d);
    float4* dst = reinterpret_cast<float4*>(xs + i * d);
    for (int l = lane; l < (d >> 2); l += 32) dst[l] = __ldg(src + l);
    if (lane == 0) ds[i] = __ldg(dense + r);
  }
}

// nb of every re-scored row back to its row; level-2 uncertain rows -> original ids (in
// place); level-2 certified pairs appended to the main pair list
__global__ void remap_uncertain_kernel(const int32_t* __restrict__ rows, int64_t nrows,
                                       const int32_t* __restrict__ sub_nb, int32_t* __restrict__ nb,
                                       int32_t* __restrict__ sub_flag, const int2* __restrict__ sub_pairs,
                                       const unsigned long long* __restrict__ sub_counts, int2* pairs,
                                       unsigned long long* pair_count) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < nrows; i += stride) nb[rows[i]] = sub_nb[i];
  const int64_t nf = static_cast<int64_t>(sub_counts[0]), np = static_cast<int64_t>(sub_counts[1]);
  for (int64_t i = t0; i < nf; i += stride) sub_flag[i] = rows[sub_flag[i]];
  for (int64_t i = t0; i < np; i += stride) {
    const int2 pr = sub_pairs[i];
    const unsigned long long j = atomicAdd(pair_count, 1ull);
    pairs[j] = make_int2(rows[pr.x], pr.y);
  }
}

// the level-2 uncertain rows become the flag list the refinement reads
__global__ void adopt_flags_kernel(const int32_t* __restrict__ sub_flag, const unsigned long long* __restrict__ sub_counts,
                                   int32_t* __restrict__ flag_rows, unsigned long long* flag_count) {
  const int64_t nf = static_cast<int64_t>(sub_counts[0]);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nf; i += stride)
    flag_rows[i] = sub_flag[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *flag_count = static_cast<unsigned long long>(nf);
}

}  // namespace

bool tc_supported(const fsil_context* c) {
  const int bn = pick_bn(c->k);
  const int kp = (c->k + bn - 1) / bn * bn;
  return c->d % 4 == 0 && c->n < (int64_t(1) << 31) && c->k >= 2 && tc_smem(bn, kp, 2) <= c->smem_optin;
}

int64_t tc_tiles(const fsil_context* c, int* tile_rows) {
  *tile_rows = BM;
  return (c->n + BM - 1) / BM;
}

void score_tc(fsil_context* c, const ScoreParams& p) {
  const bool cos = c->metric == FSIL_COSINE;
  const int bn = pick_bn(c->k);
  int ncb = (c->k + bn - 1) / bn;
  const int nkc = (c->d + BK - 1) / BK;
  const int dp = nkc * BK;
  // CTA pairs (score_tc2.cu) for streaming cluster tables: 256-column blocks, so the
  // B pieces and column tables are padded to a multiple of 256
  bool pair = false;
  {
    TcParams probe{};
    probe.nkc = nkc;
    const int nstg_ = tc_stages(bn, ncb * bn, c->smem_optin);
    const bool streaming = ncb > 1 && !(2 * nkc <= nstg_) && nkc >= nstg_;
    // (the pair kernel is a first level of one or two MMAs per K step; a single three-MMA
    // pass -- FSIL_TC_L1=3 / FSIL_TC_TWO=0 experiments -- runs on the single-CTA kernel)
    pair = streaming && pair_supported(c, probe, bn) && pair_l1(c) < 3;
    if (pair) ncb = (c->k + 255) / 256 * 2;
  }
  const int kp = ncb * bn;
  c->tc_b.ensure(2ull * kp * dp * sizeof(__half) + kp * (2 * sizeof(float) + sizeof(__half)) + sizeof(TcScale) + 96);
  __half* bh = c->tc_b.as<__half>();
  __half* bl = bh + static_cast<size_t>(kp) * dp;
  float* colbias = reinterpret_cast<float*>(bl + static_cast<size_t>(kp) * dp);
  float* lmnorm = colbias + kp;  // ||mu_k - hm_k|| (mu units, rounded up): the one-MMA level's bound
  __half* munorm = reinterpret_cast<__half*>(lmnorm + kp);
  TcScale* scale = reinterpret_cast<TcScale*>((reinterpret_cast<uintptr_t>(munorm + kp) + 31) & ~uintptr_t(31));
  float* lmmax = reinterpret_cast<float*>(scale + 1);  // max_k lmnorm (atomic max in prep_b)
  FSIL_CUDA(cudaMemsetAsync(lmmax, 0, sizeof(float), c->stream));
  TcParams tp{};
  tp.p = p;
  tp.ncb = ncb;
  tp.nkc = nkc;
  tp.colbias = colbias;
  tp.munorm = munorm;
  tp.scale = scale;
  tp.nstg = tc_stages(bn, kp, c->smem_optin);
  if (const char* e = std::getenv("FSIL_TC_NSTG")) tp.nstg = std::max(2, std::min(tp.nstg, std::atoi(e)));  // experiments
  tp.split = c->d > 128 ? 1 : 0;
  if (const char* e = std::getenv("FSIL_TC_SPLIT")) tp.split = std::atoi(e) ? 1 : 0;  // experiments
  // decoupled A slots: one cluster block, per-row ||x||^2 from the aggregation pass, and
  // room for >= 2 X stages besides the two slots
  tp.nsa = 0;
  {
    static const int dual_env = [] {
      const char* e = std::getenv("FSIL_TC_DUAL");
      return e ? std::atoi(e) : 1;
    }();
    tp.dual = dual_env;
    static const int dec_env = [] {
      const char* e = std::getenv("FSIL_TC_DECOUPLE");
      return e ? std::atoi(e) : 1;
    }();
    if (dec_env && ncb == 1 && c->xi_valid && c->agg_path == 3 && !c->X64 && tp.nstg >= 4) {
      tp.nsa = 2;
      tp.nstg -= 2;
    }
  }
  // three epilogue groups (decoupled mode at BN = 32, where the epilogue paces the kernel);
  // its six accumulator buffers must fit the 256-column allocation (no split accumulators)
  static const bool eg3_env = [] {
    const char* e = std::getenv("FSIL_TC_EG3");
    return !e || std::atoi(e) != 0;
  }();
  const bool eg3 = eg3_env && bn == 32 && tp.nsa > 0 && !tp.split;
  // unit x scale exactly where the converters take the multiply-free path (the
  // three-group kernel); its subnormal floor is bounded per row (floor_x / ||x||)
  const bool unit_ok = eg3;
  // threshold mode (see "threshold mode" above): squared Euclidean, one K chunk with a free
  // 16-column K step (D in {16, 32, 48}), several cluster blocks (A-resident tiles), the
  // label-sorted aggregation's row order for thr_kernel; FSIL_TC_THR=0 turns it off
  static const bool thr_env = [] {
    const char* e = std::getenv("FSIL_TC_THR");
    return !e || std::atoi(e) != 0;
  }();
  const bool thr = thr_env && !cos && !pair && bn == 128 && ncb > 1 && nkc == 1 && c->d % 16 == 0 && c->d <= 48 &&
                   c->agg_path == 2 && !c->X64 && tp.nstg >= 2 && c->k <= 8192;
  launch_pdl(c, prep_b_kernel, kp, 128, 0, p.stats, c->bound.as<float>(), c->xmax.as<float>(), c->k, c->d, kp, dp,
             cos, bh, bl, colbias, munorm, scale, p.abort, unit_ok, lmnorm, lmmax, thr ? c->d : 0);
  tp.lmnorm = lmnorm;
  tp.lmmax = lmmax;
  const CUtensorMap mx = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, c->X, c->d, c->n, c->d * 4ull, 32, BM);
  const CUtensorMap mh = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, bh, dp, kp, dp * 2ull, BK, bn);
  const CUtensorMap ml = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, bl, dp, kp, dp * 2ull, BK, bn);
  {
    const int64_t ntiles_ = (c->n + BM - 1) / BM;
    const bool ares_ = ncb > 1 && 2 * nkc <= tp.nstg;
    if (!ares_ && ncb > 1 && nkc >= tp.nstg) {  // streaming: per-CTA converted-A scratch
      const int64_t grid_ = std::min<int64_t>(ntiles_, c->num_sms);
      c->a_scratch.ensure(static_cast<size_t>(grid_) * nkc * kStgBytes);
      tp.ascratch = c->a_scratch.as<uint8_t>();
    }
  }
  // |dot error| <= cdot*||x||*||mu|| + floors.  Split residuals: 3 * 2^-22 relative.
  // Accumulation: tcgen05 fp32 accumulation is NOT round-to-nearest.  Measured on the
  // device (tests/test_tc_numerics.py, csrc/tc_probe.cu): each MMA (K = 16) behaves as a
  // truncating multi-term adder with 2 guard bits -- the accumulator and the 16 exact fp16
  // products are aligned to the largest exponent, each truncated toward zero to 23 + 2
  // bits below it, summed, and the sum truncated to 24 bits (that model reproduces
  // 94-100% of the probe's accumulators bit for bit; every inexact one-signed result is
  // truncated toward zero -- round 1's bias).  Worst case per MMA: (1 + 17 * 2^-2) ulps
  // (2u) of M = |accumulator| + sum |products| <= ||x~|| ||mu~|| (Cauchy-Schwarz on the
  // absolute partial sums).  Single accumulator: 3 MMAs per 16-element K step; split: the
  // main term's `steps` MMAs, the corrections (<= 2^-10 of it) separately, plus the final
  // fp32 add (u).
  const float u = 5.9604645e-8f;
  constexpr float kMmaUlp = 1.0f + 17.0f / 4.0f;
  const float steps = static_cast<float>((c->d + 15) / 16);
  tp.cdot = tp.split ? 1.05f * (12.0f + 2.0f * kMmaUlp * steps + 1.0f + 2.0f * kMmaUlp * 2.0f * steps / 512.0f) * u
                     : 1.05f * (12.0f + 2.0f * kMmaUlp * 3.0f * steps + 1.0f) * u;
  // fp64 front end: the fast pass reads the fp32 rounding of the caller's features
  // (|x32 - x| <= u|x|): +u on the dots, +2.1u on ||x||^2
  tp.exic = 8.1f;
  if (c->X64) {
    tp.cdot += 1.01f * u;
    tp.exic += 2.1f;
  }
  // ||x||^2 from the batched aggregation: fp64 over exact squares, so only its fp32
  // rounding (0.5u) remains in the bounds
  tp.xi_rows = c->xi_valid && !c->X64 ? c->xi_rows.as<double>() : nullptr;
  if (tp.xi_rows) tp.exic = 1.0f;
  // lean converters: only where the batched aggregation wrote ||x||^2 (C1/C2-like shapes);
  // the label-sorted path's ||x||^2 goes to the epilogue through the usual hand-off
  tp.lean = tp.xi_rows && c->agg_path == 3 ? 1 : 0;
  const int64_t ntiles = (c->n + BM - 1) / BM;
  static const bool prof = std::getenv("FSIL_TC_PROFILE") != nullptr;
  unsigned long long* dbg = nullptr;
  if (prof) {
    FSIL_CUDA(cudaMalloc(&dbg, 16 * sizeof(unsigned long long)));
    FSIL_CUDA(cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), c->stream));
  }
  tp.dbg = dbg;
  static const bool trace = std::getenv("FSIL_TC_TRACE") != nullptr;
  long long* trc = nullptr;
  if (trace) {
    FSIL_CUDA(cudaMalloc(&trc, 64 * 9 * sizeof(long long)));
    FSIL_CUDA(cudaMemsetAsync(trc, 0, 64 * 9 * sizeof(long long), c->stream));
  }
  tp.trace = trc;
  // top-3 / certified pairs where a full refinement row is expensive (the tiled refinement's
  // regime, K*D >= 64K) and the column halves are merged anyway (more than two blocks)
  static const bool t3_env = [] {
    const char* e = std::getenv("FSIL_TC_TOP3");
    return !e || std::atoi(e) != 0;
  }();
  const bool t3 = t3_env && bn == 128 && ncb > 2 && static_cast<int64_t>(c->k) * c->d >= 64 * 1024;
  c->pair_rows.ensure(std::max<int64_t>(c->n, 1) * sizeof(int2));
  tp.pair_rows = c->pair_rows.as<int2>();
  tp.pair_count = c->pair_count.as<unsigned long long>();  // zeroed by agg_init
  if (pair) {
    // one fp32 accumulator (512 TMEM columns hold two 256-column buffers): the correction
    // products share the main accumulator, 2 or 3 MMAs per K step in its rounding bound.
    // Two-level certificate (default): level 1 is the two-MMA pass (hx.hm + hx.lm, the
    // dropped lx.hm bounded per row by ||lx|| ||mu_k||); level 2 re-scores its uncertain rows
    // with the three-MMA kernel below.  FSIL_TC_TWO=0: one three-MMA pair pass.
    // FSIL_TC_L1 = 1 (default: one MMA per K step, hx.hm), 2 (hx.hm + hx.lm) or 3 (one
    // three-MMA pass, no second level; FSIL_TC_TWO=0 is the same)
    const int l1 = pair_l1(c);
    const bool two = l1 < 3;
    TcParams tpp = tp;
    tpp.split = 0;
    tpp.cdot = 1.05f * (12.0f + 2.0f * kMmaUlp * static_cast<float>(l1) * steps + 1.0f) * u;
    if (c->X64) tpp.cdot += 1.01f * u;
    const bool t3p = t3_env && static_cast<int64_t>(c->k) * c->d >= 64 * 1024;
    launch_tc_pair(c, mx, mh, ml, tpp, ntiles, cos, t3p, l1);
    c->tc_mmas = l1;
    if (!two) return;
    // ---- level 2
    unsigned long long nf = 0;
    FSIL_CUDA(cudaMemcpyAsync(&nf, p.flag_count, sizeof(nf), cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    const int64_t F = static_cast<int64_t>(nf);
    // (a speculation miss aborted the pass: nothing flagged; very many uncertain rows: the
    // fp64 refinement takes them all rather than a large gathered copy)
    const int64_t cap = std::max<int64_t>(1 << 16, std::min<int64_t>(c->n / 4, (int64_t(4) << 30) / (4 * c->d)));
    if (F == 0 || F > cap) return;
    c->rescored = F;
    c->sub_x.ensure(static_cast<size_t>(F) * c->d * sizeof(float));
    c->sub_i.ensure(static_cast<size_t>(F) * (3 * sizeof(int32_t) + sizeof(int2)) + 64);
    int2* sub_pairs = c->sub_i.as<int2>();
    unsigned long long* sub_counts = reinterpret_cast<unsigned long long*>(sub_pairs + F);
    int32_t* sub_dense = reinterpret_cast<int32_t*>(sub_counts + 2);
    int32_t* sub_nb = sub_dense + F;
    int32_t* sub_flag = sub_nb + F;
    float* xs = c->sub_x.as<float>();
    const unsigned g = static_cast<unsigned>(std::min<int64_t>((F + 7) / 8, static_cast<int64_t>(c->num_sms) * 8));
    gather_uncertain_kernel<<<g, 256, 0, c->stream>>>(p.X, p.dense, p.flag_rows, F, c->d, xs, sub_dense, sub_counts);
    FSIL_LAUNCHED(c);
    ScoreParams p2 = p;
    p2.X = xs;
    p2.X64 = nullptr;
    p2.dense = sub_dense;
    p2.n = F;
    p2.nb = sub_nb;
    p2.flag_rows = sub_flag;
    p2.flag_count = sub_counts;
    TcParams t2 = tp;  // the single-CTA three-MMA parameter set (split accumulators for D > 128)
    t2.p = p2;
    t2.xi_rows = nullptr;  // the gathered rows' ||x||^2: formed by the converters
    t2.exic = 8.1f;
    t2.lean = 0;
    t2.pair_rows = sub_pairs;
    t2.pair_count = sub_counts + 1;
    const int64_t nt2 = (F + BM - 1) / BM;
    const int64_t grid2 = std::min<int64_t>(nt2, c->num_sms);
    c->a_scratch.ensure(static_cast<size_t>(grid2) * nkc * kStgBytes);
    t2.ascratch = c->a_scratch.as<uint8_t>();
    const CUtensorMap mx2 = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, xs, c->d, F, c->d * 4ull, 32, BM);
    // (ms_score_kernel spans both levels: the first level's start event is kept)
    if (cos) {
      if (t3p) launch_tc<128, true, 32, 2, true>(c, mx2, mh, ml, t2, nt2, false);
      else launch_tc<128, true>(c, mx2, mh, ml, t2, nt2, false);
    } else {
      if (t3p) launch_tc<128, false, 32, 2, true>(c, mx2, mh, ml, t2, nt2, false);
      else launch_tc<128, false>(c, mx2, mh, ml, t2, nt2, false);
    }
    remap_uncertain_kernel<<<g, 256, 0, c->stream>>>(p.flag_rows, F, sub_nb, p.nb, sub_flag, sub_pairs, sub_counts,
                                                      tp.pair_rows, tp.pair_count);
    FSIL_LAUNCHED(c);
    adopt_flags_kernel<<<g, 256, 0, c->stream>>>(sub_flag, sub_counts, p.flag_rows, p.flag_count);
    FSIL_LAUNCHED(c);
    return;
  }
  c->tc_mmas = 3;
  bool thr_eg3 = false;
  if (thr) {
    c->thr_nn.ensure(static_cast<size_t>(c->k) * kThrM * sizeof(int32_t));
    c->thr_t.ensure(static_cast<size_t>(c->n) * sizeof(uint4));
    int32_t* nn = c->thr_nn.as<int32_t>();
    launch_pdl(c, nn_list_kernel, c->k, 256, (static_cast<size_t>(c->dp) + c->k) * sizeof(float), p.mu32, p.p32, c->k,
               c->d, static_cast<int>(c->dp), nn, p.abort);
    const int64_t* seg_begin = c->seg_start.as<int64_t>();
    const int64_t* seg_end = seg_begin + c->k + 1;
    const int64_t* piece_start = c->piece_start.as<int64_t>() + c->k + 2;
    const int tgrid = c->num_sms * 8;  // (blocks stride the pieces; four resident per SM)
    uint4* tt = c->thr_t.as<uint4>();
    // MMAs per K step: 1 (default: hx.hm; the dropped pieces, ~2^-11 relative, widen each
    // row's margin -- a few more two-candidate rows, a third of the tensor and operand
    // traffic) or 3 (FSIL_THR_L1=3: fp16x3)
    static const int thr_l1_env = [] { const char* e = std::getenv("FSIL_THR_L1"); return e && std::atoi(e) == 3 ? 3 : 1; }();
    tp.thr_l1 = thr_l1_env;
    if (tp.thr_l1 == 1) {
      tp.cdot = 1.05f * (12.0f + 2.0f * kMmaUlp * steps + 1.0f) * u;
      c->tc_mmas = 1;
    }
#define FSIL_THR_K(DD)                                                                                            \
  launch_pdl(c, thr_kernel<DD>, tgrid, 256, 0, p.X, c->sort_vals.as<int32_t>(), c->k, seg_begin, seg_end,       \
             piece_start, kPieceRowsTc, p.mu32, p.p32, static_cast<int>(c->dp), nn, scale, tp.cdot,           \
             tp.thr_l1 == 1 ? lmmax : nullptr, tt, p.abort)
    if (c->d == 16) FSIL_THR_K(16);
    else if (c->d == 32) FSIL_THR_K(32);
    else FSIL_THR_K(48);
#undef FSIL_THR_K
    tp.thr = c->d;
    tp.thr_t = tt;
    tp.lean = 1;  // the threshold epilogue fetches the own cluster itself; no hand-off
    // stages: a tile is one A stage for all its cluster blocks, so two or three suffice;
    // the B ring takes the rest (FSIL_THR_NB / FSIL_THR_NS: experiments)
    {
      static const int nb_env = [] { const char* e = std::getenv("FSIL_THR_NB"); return e ? std::atoi(e) : 2; }();
      static const int ns_env = [] { const char* e = std::getenv("FSIL_THR_NS"); return e ? std::atoi(e) : 4; }();
      // (ring space in hi + lo stage units: the one-MMA level fits two hi-only stages in each,
      // and the barrier arrays hold four B stages)
      int nbs = std::max(1, std::min(thr_l1_env == 1 ? 2 : 4, nb_env)), ns = std::max(2, std::min(tp.nstg, ns_env));
      while (nbs > 1 && tc_smem(bn, kp, ns, nbs) > c->smem_optin) --nbs;
      tp.nbs = nbs;
      tp.nstg = ns;
      // one-MMA level at D <= 32: a stage is box 0 alone (16 KB: the fp32 box, converted in
      // place to the hi piece), and when the whole hi-piece table (Kp x 128 B) fits beside
      // four such stages it stays resident -- no B ring, no per-block L2 reads
      // (FSIL_THR_BRES=0: ring)
      tp.astg = (tp.thr_l1 == 1 && c->d <= 32) ? kStgBytes / 2 : kStgBytes;
      static const bool bres_env = [] { const char* e = std::getenv("FSIL_THR_BRES"); return !e || std::atoi(e) != 0; }();
      const size_t tab = static_cast<size_t>(kp) * 128;
      if (bres_env && tp.thr_l1 == 1) {
        int nsr = std::min(6, std::max(2, ns_env));
        while (nsr > 2 && tc_smem(bn, kp, nsr, nbs, tp.astg, tab) > c->smem_optin) --nsr;
        if (tc_smem(bn, kp, nsr, nbs, tp.astg, tab) <= c->smem_optin) {
          tp.bres = 1;
          tp.nstg = nsr;
        }
        // three epilogue groups (three tiles in flight, one accumulator each; four converter
        // warps): resident table, D <= 32, and room for three stages + the hit slots
        // (FSIL_THR_EG3=0: two groups)
        static const bool eg3t_env = [] { const char* e = std::getenv("FSIL_THR_EG3"); return !e || std::atoi(e) != 0; }();
        if (tp.bres && eg3t_env && c->d <= 32) {
          int ns3 = 6;
          while (ns3 > 3 && tc_smem(bn, kp, ns3, nbs, tp.astg, tab, kHitSlots3) > c->smem_optin) --ns3;
          if (tc_smem(bn, kp, ns3, nbs, tp.astg, tab, kHitSlots3) <= c->smem_optin) {
            thr_eg3 = true;
            tp.nstg = ns3;
          }
        }
      }
    }
    // role rotation (see the kernel's `tid`; FSIL_TC_WSHIFT=4: issuers and producers on the
    // highest warp ids).  Measured at C4: no effect (2.79 ms either way), so off by default.
    static const int wshift_env = [] { const char* e = std::getenv("FSIL_TC_WSHIFT"); return e ? std::atoi(e) : 0; }();
    tp.wshift = (wshift_env > 0 && wshift_env % 4 == 0 && wshift_env < kThreads / 32) ? wshift_env : 0;
    c->tc_thr = 1;
    c->cand_rows.ensure(std::max<int64_t>(c->n, 1) * sizeof(int4));
    tp.cand_rows = c->cand_rows.as<int4>();
    if (thr_eg3) launch_tc<128, false, 32, 3, false, true>(c, mx, mh, ml, tp, ntiles);
    else launch_tc<128, false, 32, 2, false, true>(c, mx, mh, ml, tp, ntiles);
  }
  // K <= 24 at BN = 32: the epilogue scans only the first 16 / 24 columns
  const int kc_scan = bn == 32 && c->k <= 16 ? 16 : bn == 32 && c->k <= 24 ? 24 : 32;
  if (thr) {
  } else if (cos) {
    if (eg3 && kc_scan == 16) launch_tc<32, true, 16, 3>(c, mx, mh, ml, tp, ntiles);
    else if (eg3 && kc_scan == 24) launch_tc<32, true, 24, 3>(c, mx, mh, ml, tp, ntiles);
    else if (eg3) launch_tc<32, true, 32, 3>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 32 && kc_scan == 16) launch_tc<32, true, 16>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 32 && kc_scan == 24) launch_tc<32, true, 24>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 32) launch_tc<32, true>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 64) launch_tc<64, true>(c, mx, mh, ml, tp, ntiles);
    else if (t3) launch_tc<128, true, 32, 2, true>(c, mx, mh, ml, tp, ntiles);
    else launch_tc<128, true>(c, mx, mh, ml, tp, ntiles);
  } else {
    if (eg3 && kc_scan == 16) launch_tc<32, false, 16, 3>(c, mx, mh, ml, tp, ntiles);
    else if (eg3 && kc_scan == 24) launch_tc<32, false, 24, 3>(c, mx, mh, ml, tp, ntiles);
    else if (eg3) launch_tc<32, false, 32, 3>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 32 && kc_scan == 16) launch_tc<32, false, 16>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 32 && kc_scan == 24) launch_tc<32, false, 24>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 32) launch_tc<32, false>(c, mx, mh, ml, tp, ntiles);
    else if (bn == 64) launch_tc<64, false>(c, mx, mh, ml, tp, ntiles);
    else if (t3) launch_tc<128, false, 32, 2, true>(c, mx, mh, ml, tp, ntiles);
    else launch_tc<128, false>(c, mx, mh, ml, tp, ntiles);
  }
  if (trc) {
    long long h[64 * 9];
    FSIL_CUDA(cudaMemcpyAsync(h, trc, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    const long long t0 = h[0];
    std::fprintf(stderr, "[fsil tc trace] CTA 0, us from tile 0's X issue: tile | X-issue conv-in conv-out mma-go mma-commit epi-in epi-empty epi-done B-issue\n");
    for (int i = 0; i < 64; ++i) {
      if (!h[i * 9] && i) break;
      std::fprintf(stderr, "%3d", i);
      for (int k = 0; k < 9; ++k) std::fprintf(stderr, " %8.2f", h[i * 9 + k] ? (h[i * 9 + k] - t0) / 1965.0 : -1.0);
      std::fprintf(stderr, "\n");
    }
    cudaFree(trc);
  }
  if (dbg) {
    unsigned long long h[16];
    FSIL_CUDA(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    const char* names[14] = {"X-prod stg_empty", "B-prod op_empty", "MMA acc_empty", "MMA op_full",
                             "conv stg_full", "conv op_empty", "conv meta_empty", "epi meta_full",
                             "epi acc_full", "T prod", "T epi(w2)", "T conv(w10)", "w2 scan", "w2 finalize"};
    const double ctas = static_cast<double>(std::min<int64_t>(ntiles, c->num_sms));
    std::fprintf(stderr, "[fsil tc profile] bn=%d nstg=%d split=%d per-CTA Mcycles (waits summed over the role's warps):",
                 bn, tp.nstg, tp.split);
    for (int i = 0; i < 14; ++i) std::fprintf(stderr, " %s=%.3f", names[i], h[i] / ctas / 1e6);
    std::fprintf(stderr, "\n");
    cudaFree(dbg);
  }
}

}  // namespace fsil
