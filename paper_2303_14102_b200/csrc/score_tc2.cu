// score_tc2.cu -- K3 on CTA pairs: tcgen05.mma.cta_group::2 for large cluster tables.
//
// Same job as score_tc.cu's streaming mode -- nominate each row's neighbour cluster from
// the split-precision ("fp16x3") dots x . mu_k with a certified bound; replaces the
// neighbour loop of score_range (squared_euclidean.cpp:96-103, cosine.cpp:105-112) -- but
// the MMAs are 256 x 256 x 16 over the two CTAs of a cluster (one TPC).  The single-CTA
// kernel's 128 x 128 x 16 MMA reads 8 KB of shared memory per 64 tensor cycles (all of an
// SM's shared-memory bandwidth) and, streaming a 4096-column table, pulls 64 KB of
// operands from L2 per 12 MMAs.  Here each CTA holds its own 128 rows of A and its own 128
// of the block's 256 B columns: per SM an MMA reads 8 KB per 128 cycles and the L2
// operand traffic per flop halves.
//
// Roles per CTA (640 threads, 20 warps; registers as score_tc.cu):
//   warp 0      X producer: TMA of this CTA's 128 rows on the first pass over a tile; on
//               the later cluster blocks, cta_group::2 tensor copies of the converted
//               chunks back from this CTA's L2-resident scratch, completing on the
//               LEADER's a_full barrier
//   warp 1      TMEM: cta_group::2 allocation of 512 columns (two 256-column fp32
//               accumulators); in the leader CTA, lane 0 issues every MMA of the pair
//   warp 2      B producer: this CTA's 128 columns (hi, lo) of each 256-column block,
//               completing on the leader's b_full barrier
//   warps 4-11  epilogue: two groups of four split each block's eight 32-column chunks;
//               keys, running top-3, certification (certify_row, score_tc.cuh)
//   warps 12-19 converters: fp32 -> fp16 hi/lo in place (2 threads per row), store of the
//               converted chunk to the scratch, one arrival per chunk on the leader
//
// Cross-CTA protocol.  Barriers the MMA issuer waits on live in the leader (rank 0):
// a_full (2 arrivals: one per CTA; reload passes add the bytes of both CTAs' copies),
// b_full (the leader's expect_tx covers both CTAs' B bytes) and acc_empty (8 epilogue
// warps of each CTA).  The MMA commits multicast to both CTAs' stg_empty, b_empty and
// acc_full.  Remote arrivals are release.cluster; the issuer's waits acquire.cluster.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "score_tc.cuh"

namespace fsil {
namespace tc {
namespace {

constexpr int kPairN = 256;                // MMA N: cluster columns per block
constexpr int kHalfN = 128;                // B columns held by each CTA
constexpr int kBPiece = kHalfN * 128;      // one B piece (hi or lo) per stage per CTA: 16 KB
constexpr uint32_t kPairCols = 512;        // TMEM columns: two 256-column accumulators
constexpr int kEpi0 = 4, kConv0 = 12;
constexpr int kScanG = 4;  // epilogue filter group (keys)
constexpr int kXBox = BM * 128;            // one X box: 128 rows x 32 fp32 columns (16 KB)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;\n" : "=r"(r));
  return r;
}
// shared::cluster address of the same object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(caddr) : "memory");
}
// arrival on a barrier of another CTA of the cluster without a cluster-scope release: for
// signals that publish no memory (the epilogue's TMEM reads have completed -- tcgen05.wait::ld
// -- before it frees the accumulator), the release fence would only add latency
__device__ __forceinline__ void mbar_arrive_remote(uint32_t caddr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(caddr) : "memory");
}
// tx bytes expected on a local barrier without arriving (the leader's reload items)
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// `count` arrivals at once on a local barrier (the leader arrives for both CTAs of the pair
// on reload items: neither CTA wrote the stage with generic stores, so the peer's arrival
// would publish nothing and its cluster-scope release fence is pure latency)
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
// wait with cluster-scope acquire: the phase may have been completed by the peer CTA
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
        : "memory");
  } while (!ok);
}
// Optional wait profiling (FSIL_TC_PROFILE): cycles spent in a wait, added to dbg[slot]
#define PW(slot, call)                                                                   \
  do {                                                                                   \
    if (dbg) {                                                                           \
      const long long t0__ = clock64();                                                  \
      call;                                                                              \
      atomicAdd(dbg + (slot), static_cast<unsigned long long>(clock64() - t0__));       \
    } else {                                                                             \
      call;                                                                              \
    }                                                                                    \
  } while (0)

// 2-D tensor copy of the pair (cta_group::2): lands in this CTA's shared memory, the
// transaction bytes complete on the barrier at cluster address `bar_caddr` (the leader's)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_caddr, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_caddr)
      : "memory");
}
// L2 eviction-priority policies for the tensor copies: the X stream is read once
// (evict_first), the converted-A scratch and the B pieces are re-read every cluster block
// (evict_last), so X does not push them out of L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair_hint(void* dst, const CUtensorMap* map, uint32_t bar_caddr, int c0,
                                                      int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_caddr), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(
                   reinterpret_cast<uint64_t>(dst)),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}

// 2-D tensor store from this CTA's shared memory (bulk group: commit here, the caller waits)
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int c0, int c1,
                                                  uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(pol)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}

template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(smem_dst)),
               "n"(NCOLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(NCOLS));
}
// D[tmem of both CTAs] (+)= A[256 x 16: 128 rows per CTA] * B[256 x 16: 128 columns per CTA]^T
__device__ __forceinline__ void mma_f16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this offset in every CTA of `mask` once the issued MMAs retire
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// one lane of a converged warp (the issuing lane of a warp-wide loop)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// Shared memory (identical offsets in both CTAs: the MMA addresses the peer's operands
// through the leader's descriptors)
struct PairSmem {
  static size_t bytes(int ns, int nb, int nx) {
    return 1024 + static_cast<size_t>(ns) * kStgBytes + static_cast<size_t>(nb) * 2 * kBPiece +
           static_cast<size_t>(nx) * kXBox + 64 * 8 + 4 * BM * 8 + 10 * BM * 4 + 2 * BM * 4 + 4 * BM * 4 + 64;
  }
};

// TWO: the first level of a two-level certificate -- two MMAs per K step, hx.hm + hx.lm
// (the x pieces' low half dropped; its contribution is bounded per row by ||lx|| ||mu_k||,
// lx = x~ - hx exact in fp32), A operands of 16 KB per chunk.  Rows it cannot certify are
// re-scored at three-MMA precision (score_tc.cu, level 2).
// L1 = 1: the first level is a single MMA per K step, hx.hm: the dropped hx.lm is bounded per
// column by ||hx|| ||mu_k - hm_k|| (prep_b's lmnorm table), and only hm is loaded for B.
template <bool COS, bool T3, int L1>
__global__ void __launch_bounds__(kThreads, 1)
    score_tc_pair_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_bh,
                         const __grid_constant__ CUtensorMap tmap_bl, const __grid_constant__ CUtensorMap tmap_scr,
                         const __grid_constant__ CUtensorMap tmap_scst, TcParams tp, int64_t ntiles, int ns, int nb,
                         int nx) {
  static_assert(L1 == 1 || L1 == 2, "the pair kernel is the first level of the two-level certificate");
  constexpr int BCH = L1 == 1 ? 2 : 1;  // K chunks per B stage (hm only: two fit a stage)
  constexpr int ACH = 2;                // K chunks per A stage (hx only: two fit a stage)
  griddep_wait();           // (PDL) prep_b's operands and every earlier phase are visible
  if (*tp.p.abort) return;  // K speculation missed: the call is repeated (both CTAs return)
  const ScoreParams& p = tp.p;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int ncb = tp.ncb, nkc = tp.nkc;
  const int64_t nst = (ntiles + 1) / 2;  // super-tiles of 256 rows
  const int64_t cid = cluster_id_x(), ncl = cluster_count_x();
  constexpr uint32_t kIdesc = idesc_f16_f32(256, kPairN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stg = base;                               // [ns][2 x 16 KB]: A items (hx of two K chunks)
  uint8_t* bring = stg + ns * kStgBytes;             // [nb][2 x 16 KB]: B (this CTA's 128 columns)
  uint8_t* xst = bring + nb * 2 * kBPiece;           // [nx][16 KB]: X fp32 boxes (32 columns)
  uint64_t* bars = reinterpret_cast<uint64_t*>(xst + nx * kXBox);
  uint64_t* stg_empty = bars;        // [ns <= 8] local: A stage free (multicast MMA commit)
  uint64_t* a_full = bars + 8;       // [ns] leader: both CTAs' reloaded chunks landed
  uint64_t* b_full = bars + 16;      // [nb <= 8] leader: B of both CTAs
  uint64_t* b_empty = bars + 24;     // [nb] local (multicast commit)
  uint64_t* acc_full = bars + 32;    // [2] local (multicast commit)
  uint64_t* acc_empty = bars + 34;   // [2] leader: 8 epilogue warps x 2 CTAs
  uint64_t* meta_full = bars + 36;   // [2] local
  uint64_t* meta_empty = bars + 38;  // [2] local
  uint64_t* scr_ready = bars + 40;   // [2] local: a tile's converted chunks are in scratch buffer b
  uint64_t* scr_free = bars + 42;    // [2] local: the issuer is past every reload of buffer b's tile
  uint64_t* xs_full = bars + 44;     // [nx <= 4] local: X box landed
  uint64_t* xs_empty = bars + 48;    // [nx] local: X box converted and stored
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 52);
  double* meta_xi = reinterpret_cast<double*>(bars + 64);    // [2][2][BM]
  float* part = reinterpret_cast<float*>(meta_xi + 4 * BM);  // [2][5][BM]
  int* meta_own = reinterpret_cast<int*>(part + 10 * BM);     // [2][BM]
  float* meta_lx = reinterpret_cast<float*>(meta_own + 2 * BM);  // [2][2][BM] ||lx||^2 halves

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA's scratch: [2 buffers][nkc chunks][BM rows][64 fp16], rows of the 2-D map
  const int64_t scr_row0 = static_cast<int64_t>(blockIdx.x) * 2 * nkc * BM;
  const int nbx = (p.d + 31) / 32;  // X boxes (32 fp32 columns) per tile
  const TcScale sc = *tp.scale;
  unsigned long long* const dbg = tp.dbg;
  const long long t_begin = dbg ? clock64() : 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(stg_empty + i, 1);
      mbar_init(a_full + i, 2);
    }
    for (int i = 0; i < nb; ++i) {
      mbar_init(b_full + i, 1);
      mbar_init(b_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(acc_full + i, 1);
      mbar_init(acc_empty + i, 16);
      mbar_init(meta_full + i, 8);
      mbar_init(meta_empty + i, 4);
      mbar_init(scr_ready + i, 1);
      mbar_init(scr_free + i, 1);
    }
    for (int i = 0; i < nx; ++i) {
      mbar_init(xs_full + i, 1);
      mbar_init(xs_empty + i, 1);
    }
    fence_barrier_init();
    prefetch_tmap(&tmap_x);
    prefetch_tmap(&tmap_bh);
    prefetch_tmap(&tmap_bl);
    prefetch_tmap(&tmap_scr);
    prefetch_tmap(&tmap_scst);
  }
  if (warp == 1) tmem_alloc_pair<kPairCols>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < kEpi0) {
    setmaxnreg_dec<64>();
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------ A producer
      // every pass over a tile (all ncb cluster blocks) reloads its converted chunks from
      // this CTA's scratch buffer, two chunks per stage, completing on the leader's a_full
      uint32_t n1 = 0, ntl = 0;
      const uint64_t pol_keep = l2_policy_evict_last();
      for (int64_t st = cid; st < nst; st += ncl, ++ntl) {
        const int64_t srow = scr_row0 + static_cast<int64_t>(ntl & 1) * nkc * BM;
        PW(5, mbar_wait(scr_ready + (ntl & 1), (ntl >> 1) & 1));
        fence_proxy_async_global();
        for (int cb = 0; cb < ncb; ++cb) {
          for (int kc = 0; kc < nkc; kc += ACH, ++n1) {
            const int s1 = static_cast<int>(n1 % ns);
            PW(4, mbar_wait(stg_empty + s1, ((n1 / ns) & 1) ^ 1));  // (multicast MMA commit)
            const uint32_t af = mapa_u32(smem_u32(a_full + s1), 0);
            const int nch = min(ACH, nkc - kc);
            if (leader) mbar_expect_tx(a_full + s1, 2 * nch * kABytes);
            for (int h = 0; h < nch; ++h)
              tma_load_2d_pair_hint(stg + s1 * kStgBytes + h * kABytes, &tmap_scr, af, 0,
                                    static_cast<int>(srow + (kc + h) * BM), pol_keep);
            if (leader) mbar_arrive_cnt(a_full + s1, 2);
          }
        }
      }
    } else if (warp == 3 && lane == 0) {
      // ------------------------------------------------------------ X producer
      // this CTA's 128 rows of each tile, one 32-column box per stage; runs up to the X ring
      // ahead, so the next tile's rows stream in while the current tile is scored
      uint32_t nxb = 0;
      const uint64_t pol_x = l2_policy_evict_first();
      for (int64_t st = cid; st < nst; st += ncl) {
        const int row0 = static_cast<int>(st * 2 * BM + rank * BM);
        for (int bx = 0; bx < nbx; ++bx, ++nxb) {
          const int sx = static_cast<int>(nxb % nx);
          mbar_wait(xs_empty + sx, ((nxb / nx) & 1) ^ 1);
          mbar_arrive_expect_tx(xs_full + sx, kXBox);
          tma_load_2d_hint(xst + sx * kXBox, &tmap_x, xs_full + sx, bx * 32, row0, pol_x);
        }
      }
    } else if (warp == 2 && lane == 0) {
      // ------------------------------------------------------------ B producer
      uint32_t n2 = 0;
      const uint64_t pol_b = l2_policy_evict_last();
      for (int64_t st = cid; st < nst; st += ncl) {
        for (int cb = 0; cb < ncb; ++cb) {
          for (int kc = 0; kc < nkc; kc += BCH, ++n2) {
            const int sb = static_cast<int>(n2 % nb);
            uint8_t* bs = bring + sb * 2 * kBPiece;
            PW(6, mbar_wait(b_empty + sb, ((n2 / nb) & 1) ^ 1));
            const uint32_t bf = mapa_u32(smem_u32(b_full + sb), 0);
            const int col = cb * kPairN + static_cast<int>(rank) * kHalfN;
            if (L1 == 1) {  // hm of two consecutive chunks per stage (B lookahead doubles)
              const int nch = min(2, nkc - kc);
              if (leader) mbar_arrive_expect_tx(b_full + sb, nch * 2 * kBPiece);
              for (int h = 0; h < nch; ++h)
                tma_load_2d_pair_hint(bs + h * kBPiece, &tmap_bh, bf, (kc + h) * BK, col, pol_b);
            } else {
              if (leader) mbar_arrive_expect_tx(b_full + sb, 4 * kBPiece);
              tma_load_2d_pair_hint(bs, &tmap_bh, bf, kc * BK, col, pol_b);
              tma_load_2d_pair_hint(bs + kBPiece, &tmap_bl, bf, kc * BK, col, pol_b);
            }
          }
        }
      }
    } else if (warp == 1 && leader) {
      // ------------------------------------------------------------ MMA issuer (the pair's)
      // The whole warp runs the loop (every value on it warp-uniform, so descriptors live in
      // uniform registers) and one elected lane issues: a single-thread loop paid a
      // uniform-register waterfall per MMA and could not keep the tensor pipe fed.
      unsigned long long* const dbg = lane == 0 ? tp.dbg : nullptr;
      const bool nomma = tp.dbg && tp.dbg[15] != 0;  // FSIL_TC_PROFILE=2 diagnostic: the pipeline without MMAs
      uint32_t na = 0;
      // ring positions advance incrementally (no runtime division on the issue path)
      int s1 = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      const int nkfull = p.d / BK;  // full 64-wide K chunks
      const uint64_t da0 = desc_k_sw128(smem_u32(stg)), db0 = desc_k_sw128(smem_u32(bring));
      uint32_t ntl = 0;
      for (int64_t st = cid; st < nst; st += ncl, ++ntl) {
        for (int cb = 0; cb < ncb; ++cb, ++na) {
          const int ab = static_cast<int>(na & 1);
          PW(0, mbar_wait(acc_empty + ab, ((na >> 1) & 1) ^ 1));
          tc_fence_after();
          const uint32_t d = tmem_base + ab * kPairN;
          constexpr int ach = ACH;  // chunks per A item
          const long long tcb0 = dbg ? clock64() : 0;
          for (int kc0 = 0; kc0 < nkc; kc0 += ach) {
            const long long tit0 = dbg ? clock64() : 0;
            if (L1 == 1 && kc0 + 2 <= nkfull) {
              // the steady state: a reload item of two full chunks against the B stage of the
              // same two chunks -- two waits, eight MMAs, two commits, straight-line
              PW(1, mbar_wait(a_full + s1, pa));
              PW(2, mbar_wait(b_full + sb, pb));
              tc_fence_after();
              if (elect_one()) {
                const uint64_t da = da0 + static_cast<uint32_t>(s1 * (kStgBytes >> 4)),
                               db = db0 + static_cast<uint32_t>(sb * (2 * kBPiece >> 4));
                if (!nomma) {
#pragma unroll
                  for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                      mma_f16_pair(d, da + h * (kABytes >> 4) + 2 * ks, db + h * (kBPiece >> 4) + 2 * ks, kIdesc,
                                   (h | ks | kc0) ? 1u : 0u);
                }
                mma_commit_pair(b_empty + sb, 0x3);
                mma_commit_pair(stg_empty + s1, 0x3);
              }
              __syncwarp();
              if (++sb == nb) {
                sb = 0;
                pb ^= 1u;
              }
              if (++s1 == ns) {
                s1 = 0;
                pa ^= 1u;
              }
              if (dbg) atomicAdd(dbg + 12, static_cast<unsigned long long>(clock64() - tit0));
              continue;
            }
            // (the tensor copies' completions make their bytes visible to the async proxy
            // through the barrier itself: CTA-scope waits)
            PW(1, mbar_wait(a_full + s1, pa));
            const int nch = min(ach, nkc - kc0);
            for (int h = 0; h < nch; ++h) {
              const int kc = kc0 + h;
              const int bh = BCH == 2 ? (kc & 1) : 0;  // chunk's half of the B stage
              if (bh == 0) PW(2, mbar_wait(b_full + sb, pb));
              tc_fence_after();
              const int rem = p.d - kc * BK;
              const int nks = rem >= BK ? 4 : (rem + 15) / 16;
              const uint64_t dah = desc_k_sw128(smem_u32(stg + s1 * kStgBytes + h * kABytes)),
                             dal = dah + (kABytes >> 4);
              const uint64_t dbh = desc_k_sw128(smem_u32(bring + sb * 2 * kBPiece + bh * kBPiece)),
                             dbl = dbh + (kBPiece >> 4);
              const bool b_done = BCH == 1 || bh == 1 || kc + 1 == nkc;  // the B stage's last chunk
              const bool a_done = h + 1 == nch;                          // the A item's last chunk
              if (elect_one()) {
                const long long ti0 = dbg ? clock64() : 0;
                if (nomma) {
                } else if (nks == 4) {
#pragma unroll
                  for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
                    mma_f16_pair(d, dah + 2 * ks, dbh + 2 * ks, kIdesc, acc0);
                    if (L1 > 1) mma_f16_pair(d, dah + 2 * ks, dbl + 2 * ks, kIdesc, 1u);
                    if (L1 > 2) mma_f16_pair(d, dal + 2 * ks, dbh + 2 * ks, kIdesc, 1u);
                  }
                } else {
                  for (int ks = 0; ks < nks; ++ks) {
                    const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
                    mma_f16_pair(d, dah + 2 * ks, dbh + 2 * ks, kIdesc, acc0);
                    if (L1 > 1) mma_f16_pair(d, dah + 2 * ks, dbl + 2 * ks, kIdesc, 1u);
                    if (L1 > 2) mma_f16_pair(d, dal + 2 * ks, dbh + 2 * ks, kIdesc, 1u);
                  }
                }
                if (b_done) mma_commit_pair(b_empty + sb, 0x3);
                if (a_done) mma_commit_pair(stg_empty + s1, 0x3);
                if (dbg) atomicAdd(dbg + 11, static_cast<unsigned long long>(clock64() - ti0));
              }
              __syncwarp();
              if (b_done && ++sb == nb) {
                sb = 0;
                pb ^= 1u;
              }
            }
            if (++s1 == ns) {
              s1 = 0;
              pa ^= 1u;
            }
            if (dbg) atomicAdd(dbg + 12, static_cast<unsigned long long>(clock64() - tit0));
          }
          if (elect_one()) mma_commit_pair(acc_full + ab, 0x3);
          __syncwarp();
          if (dbg) atomicAdd(dbg + 13, static_cast<unsigned long long>(clock64() - tcb0));
        }
        // every reload of this tile's scratch buffer has landed (its a_full waits are
        // behind us): both CTAs' converters may overwrite the buffer with the tile after next
        if (elect_one()) {
          mbar_arrive(scr_free + (ntl & 1));
          mbar_arrive_remote(mapa_u32(smem_u32(scr_free + (ntl & 1)), 1));
        }
        __syncwarp();
      }
      if (dbg) atomicAdd(dbg + 3, static_cast<unsigned long long>(clock64() - t_begin));
    }
  } else if (warp >= kConv0) {
    setmaxnreg_dec<72>();
    // ------------------------------------------------------------ converters
    // One X box (32 fp32 columns x 128 rows) at a time, two threads per row (16 columns
    // each): scale (exact), fp16 hx, the residual lx = x~ - hx (exact) into ||lx||^2; hx is
    // written in place as a compact [128 rows][64 B] half chunk and tensor-stored to this
    // CTA's scratch buffer of the tile.  Converting runs a tile ahead of the MMAs (double-
    // buffered scratch): no pass over a tile waits on HBM or on the conversion.
    const int tl = threadIdx.x - kConv0 * 32;
    const int r = tl & (BM - 1), hq = tl >> 7;
    const int sw = r & 7;
    const float2 sx2 = make_float2(sc.sx, sc.sx), neg1 = make_float2(-1.f, -1.f);
    const uint64_t pol_keep = l2_policy_evict_last();
    uint32_t nxb = 0, nt = 0;
    for (int64_t st = cid; st < nst; st += ncl, ++nt) {
      const int64_t row = st * 2 * BM + rank * BM + r;
      const int own = (hq == 0 && row < p.n) ? __ldg(p.dense + row) : -1;
      const int b = static_cast<int>(nt & 1);
      const int64_t srow = scr_row0 + static_cast<int64_t>(b) * nkc * BM;
      double xi = 0.0;
      float lx2 = 0.0f;  // sum of lx^2 (exact residuals; tiny, fp32 sum + margin)
      for (int bx = 0; bx < nbx; ++bx, ++nxb) {
        const int sx = static_cast<int>(nxb % nx);
        if (tl == 0) PW(9, mbar_wait(xs_full + sx, (nxb / nx) & 1));
        else mbar_wait(xs_full + sx, (nxb / nx) & 1);
        uint8_t* xb = xst + sx * kXBox;
        float4 f[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) f[u] = *reinterpret_cast<const float4*>(xb + r * 128 + (((4 * hq + u) ^ sw) << 4));
        named_bar_sync(5, 256);  // every read of the box precedes the in-place writes
        const float v[16] = {f[0].x, f[0].y, f[0].z, f[0].w, f[1].x, f[1].y, f[1].z, f[1].w,
                             f[2].x, f[2].y, f[2].z, f[2].w, f[3].x, f[3].y, f[3].z, f[3].w};
        if (!tp.xi_rows) {  // ||x||^2: fp32 blocks of 8 (error <= 8u each), fp64 across blocks
#pragma unroll
          for (int blk = 0; blk < 2; ++blk) {
            float2 bs = make_float2(0.f, 0.f);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 ve = make_float2(v[8 * blk + 2 * e], v[8 * blk + 2 * e + 1]);
              bs = __ffma2_rn(ve, ve, bs);
            }
            xi += static_cast<double>(bs.x + bs.y);
          }
        }
        uint32_t hw[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {  // packed f32x2: scale (exact), hi, residual (exact)
          const float2 xx = __fmul2_rn(make_float2(v[2 * e], v[2 * e + 1]), sx2);
          const __half2 h = __float22half2_rn(xx);
          const float2 res = __ffma2_rn(__half22float2(h), neg1, xx);
          lx2 = fmaf(res.x, res.x, fmaf(res.y, res.y, lx2));
          hw[e] = *reinterpret_cast<const uint32_t*>(&h);
        }
        uint8_t* hrow = xb + r * 64 + hq * 32;
        *reinterpret_cast<uint4*>(hrow) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(hrow + 16) = make_uint4(hw[4], hw[5], hw[6], hw[7]);
        fence_proxy_async_smem();
        named_bar_sync(5, 256);
        if (tl == 0) {
          // the buffer last held the tile before last: the issuer must be past its reloads
          if (bx == 0 && nt >= 2) PW(14, mbar_wait(scr_free + b, ((nt >> 1) & 1) ^ 1));
          tma_store_2d_hint(&tmap_scst, xb, (bx & 1) * 32, static_cast<int>(srow + (bx >> 1) * BM), pol_keep);
          bulk_wait_read();
          mbar_arrive(xs_empty + sx);
        }
      }
      if (tl == 0) {  // this tile's chunks are all in global memory
        bulk_wait_all();
        mbar_arrive(scr_ready + b);
      }
      // ||x||^2 halves, ||lx||^2 halves and the own cluster to the epilogue
      const int tb = nt & 1;
      mbar_wait(meta_empty + tb, ((nt >> 1) & 1) ^ 1);
      meta_xi[(tb * 2 + hq) * BM + r] = xi;
      meta_lx[(tb * 2 + hq) * BM + r] = lx2;
      if (hq == 0) meta_own[tb * BM + r] = own;
      __syncwarp();
      if (lane == 0) mbar_arrive(meta_full + tb);
    }
  } else {
    // ------------------------------------------------------------ epilogue (8 warps)
    setmaxnreg_inc<136>();
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int grp = (warp - kEpi0) >> 2;
    uint32_t na = 0, nt = 0;
    constexpr int NQ = kPairN / 32;
    for (int64_t st = cid; st < nst; st += ncl, ++nt) {
      const int tb = nt & 1;
      const int64_t row = st * 2 * BM + rank * BM + r;
      const bool valid = row < p.n;
      const double xi_g = (tp.xi_rows && valid) ? __ldg(tp.xi_rows + row) : 0.0;
      if (threadIdx.x == 32 * kEpi0) PW(8, mbar_wait(meta_full + tb, (nt >> 1) & 1));
      else mbar_wait(meta_full + tb, (nt >> 1) & 1);
      const int own = meta_own[tb * BM + r];
      const double xi64 = tp.xi_rows ? xi_g : meta_xi[(tb * 2) * BM + r] + meta_xi[(tb * 2 + 1) * BM + r];
      const float xi = static_cast<float>(xi64);
      const float xn = COS ? 0.0f : sqrtf(xi);
      const float rnf = COS ? rsqrtf(xi) : 0.0f;
      const float rowm = COS ? -(sc.smul * rnf) : -2.0f * sc.smul;
      // ||lx|| / ||x~|| (the dropped piece, relative to the row; fp32 sums of squares of
      // numbers ~2^-11 |x| carry < 1e-4 relative error: x 1.001 margin; rsqrt <= 2.2u)
      const float lx_rel =
          sqrtf(meta_lx[(tb * 2) * BM + r] + meta_lx[(tb * 2 + 1) * BM + r]) * rsqrtf(xi) / sc.sx * 1.001f;
      float b1 = INFINITY, b2 = INFINITY, b3 = INFINITY;
      int arg = -1, arg2 = -1;
      // one 32-column chunk: ranking keys (own column excluded), running top-2 / top-3.
      // The ALU pipe (compares, selects, min/max: half rate) bounds this loop, so the chunk
      // goes in groups of kScanG keys: the group's minimum against the running threshold
      // (b3 -- b2 without T3) and the full update only when some row of the warp has a key
      // below it.  Skipping is exact: a key >= the threshold changes none of b1..b3 / args.
      auto scan32 = [&](const uint32_t(&v)[32], int k0) {
        const int ownrel = own - k0;
        int argc = -1;
        const float4* cb4 = reinterpret_cast<const float4*>(tp.colbias + k0);
        float bj[32];
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 bias = __ldg(cb4 + j4);
          bj[4 * j4] = bias.x;
          bj[4 * j4 + 1] = bias.y;
          bj[4 * j4 + 2] = bias.z;
          bj[4 * j4 + 3] = bias.w;
        }
#pragma unroll
        for (int g = 0; g < 32 / kScanG; ++g) {
          float m[kScanG];
#pragma unroll
          for (int e = 0; e < kScanG; ++e) m[e] = fmaf(__uint_as_float(v[g * kScanG + e]), rowm, bj[g * kScanG + e]);
          float gmin = m[0];
#pragma unroll
          for (int e = 1; e < kScanG; ++e) gmin = fminf(gmin, m[e]);
          if (!__any_sync(0xffffffffu, gmin < (T3 ? b3 : b2))) continue;
#pragma unroll
          for (int e = 0; e < kScanG; ++e) {
            const int j = g * kScanG + e;
            const float mm = j == ownrel ? INFINITY : m[e];
            const bool lt = mm < b1;  // strict: the lowest index keeps ties
            if (T3) {
              const bool lt2 = mm < b2;
              arg2 = lt ? arg : (lt2 ? k0 + j : arg2);
              arg = lt ? k0 + j : arg;
              b3 = fminf(b3, fmaxf(b2, mm));
            } else {
              argc = lt ? j : argc;
            }
            b2 = fminf(b2, fmaxf(b1, mm));
            b1 = fminf(b1, mm);
          }
        }
        if (!T3 && argc >= 0) arg = k0 + argc;
      };
      for (int cb = 0; cb < ncb; ++cb, ++na) {
        const int ab = static_cast<int>(na & 1);
        if (threadIdx.x == 32 * kEpi0) PW(7, mbar_wait(acc_full + ab, (na >> 1) & 1));
        else mbar_wait(acc_full + ab, (na >> 1) & 1);
        tc_fence_after();
        const uint32_t tb0 = tmem_base + ab * kPairN + (static_cast<uint32_t>(quad * 32) << 16);
#pragma unroll 1
        for (int q = grp; q < NQ; q += 4) {  // this group's chunks q and q + 2, one TMEM wait
          uint32_t v[32], w[32];
          tmem_ld32_issue(tb0 + q * 32, v);
          tmem_ld32_issue(tb0 + (q + 2) * 32, w);
          tmem_ld_wait2(v, w);
          scan32(v, cb * kPairN + q * 32);
          scan32(w, cb * kPairN + (q + 2) * 32);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(mapa_u32(smem_u32(acc_empty + ab), 0));
      }
      // ---- merge the two column halves (group 1 -> smem -> group 0)
      float* pt = part + tb * 5 * BM;
      if (grp == 1) {
        pt[0 * BM + r] = b1;
        pt[1 * BM + r] = b2;
        pt[2 * BM + r] = __int_as_float(arg);
        pt[3 * BM + r] = b3;
        pt[4 * BM + r] = __int_as_float(arg2);
      }
      named_bar_sync(1, 256);
      if (grp == 1) continue;
      const float c1 = pt[0 * BM + r], c2 = pt[1 * BM + r];
      const int a2 = __float_as_int(pt[2 * BM + r]);
      if (T3) {
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
      // group 0 has read the partials and the meta slot: both may be reused
      __syncwarp();
      if (lane == 0) mbar_arrive(meta_empty + tb);
      if (valid)
        certify_row<COS, T3>(tp, sc, row, own, xi, xn, rnf, b1, b2, b3, arg, arg2,
                                       arg >= 0 ? __half2float(__ldg(tp.munorm + arg)) : 1.0f,
                                       arg2 >= 0 ? __half2float(__ldg(tp.munorm + arg2)) : 1.0f, lx_rel,
                                       L1 == 1 && arg >= 0 ? __ldg(tp.lmnorm + arg) : 0.0f,
                                       L1 == 1 && arg2 >= 0 ? __ldg(tp.lmnorm + arg2) : 0.0f,
                                       L1 == 1 ? __ldg(tp.lmmax) : 0.0f);
    }
  }

  tc_fence_before();
  cluster_sync_all();  // both CTAs done with the pair's TMEM and barriers
  if (warp == 1) tmem_dealloc_pair<kPairCols>(tmem_base);
}

}  // namespace

bool pair_supported(const fsil_context* c, const TcParams& tp, int bn) {
  static const bool env = [] {
    const char* e = std::getenv("FSIL_TC_PAIR");
    return !e || std::atoi(e) != 0;
  }();
  // streaming regime only (several 256-column blocks, a tile's chunks too many to keep),
  // an even grid of one CTA per SM
  const int ncb2 = (c->k + kPairN - 1) / kPairN;
  return env && bn == 128 && ncb2 >= 2 && tp.nkc >= 3 && c->num_sms >= 2 && !c->X64 &&
         PairSmem::bytes(3, 3, 1) <= c->smem_optin;
}

void launch_tc_pair(fsil_context* c, const CUtensorMap& mx, const CUtensorMap& mh, const CUtensorMap& ml,
                    TcParams tp, int64_t ntiles, bool cos, bool t3, int l1) {
  if (l1 < 1 || l1 > 2) fail(FSIL_ERR_INTERNAL, "pair kernel: first level of 1 or 2 MMAs per K step");
  // stages: A (two reloaded chunks) and B rings of 32 KB, X boxes of 16 KB.  Measured (C5,
  // 1M rows, Mcycles per CTA): 3/3/1 6.62, 3/2/2 7.32, 2/3/2 7.85 -- the converters run a
  // tile ahead and need no X lookahead; the MMA needs both operand rings deep
  int ns = 3, nb = 3, nx = 1;
  if (const char* e = std::getenv("FSIL_TC_PAIR_NB")) nb = std::max(2, std::min(8, std::atoi(e)));  // experiments
  if (const char* e = std::getenv("FSIL_TC_PAIR_NS")) ns = std::max(2, std::min(8, std::atoi(e)));
  if (const char* e = std::getenv("FSIL_TC_PAIR_NX")) nx = std::max(1, std::min(4, std::atoi(e)));
  while (PairSmem::bytes(ns, nb, nx) > c->smem_optin && ns > 2) --ns;
  while (PairSmem::bytes(ns, nb, nx) > c->smem_optin && nb > 2) --nb;
  while (PairSmem::bytes(ns, nb, nx) > c->smem_optin && nx > 1) --nx;
  tp.ncb = (c->k + kPairN - 1) / kPairN;
  // (Measured and removed: a fused exact pass in the converters -- the post pass 45 -> 11 ms
  // but the kernel 636 -> 685 ms, fp64 table reads competing with the operand stream in L2.
  // DESIGN.md 4.5.)
  const int grid = static_cast<int>(std::max<int64_t>(2, std::min<int64_t>(2 * ((ntiles + 1) / 2), c->num_sms & ~1)));
  // scratch: per CTA two buffers (the tile being scored, the next being converted) of nkc
  // chunks x 128 rows x 64 fp16 -- a 2-D tensor of 128-byte rows, reloaded in 64 x 128
  // boxes with the 128-byte swizzle the MMA descriptors expect, stored by the converters
  // in unswizzled 32 x 128 half chunks
  const uint64_t srows = static_cast<uint64_t>(grid) * 2 * tp.nkc * BM;
  c->a_scratch.ensure(srows * 128);
  tp.ascratch = c->a_scratch.as<uint8_t>();
  const CUtensorMap mscr = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, tp.ascratch, 64, srows, 128, 64, BM,
                                       CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap mscst = make_map_2d(CU_TENSOR_MAP_DATA_TYPE_FLOAT16, tp.ascratch, 64, srows, 128, 32, BM,
                                        CU_TENSOR_MAP_SWIZZLE_NONE);
  const size_t smem = PairSmem::bytes(ns, nb, nx);
#define FSIL_PAIR_K(L) (cos ? (t3 ? score_tc_pair_kernel<true, true, L> : score_tc_pair_kernel<true, false, L>) \
                           : (t3 ? score_tc_pair_kernel<false, true, L> : score_tc_pair_kernel<false, false, L>))
  auto kern = l1 == 1 ? FSIL_PAIR_K(1) : FSIL_PAIR_K(2);
#undef FSIL_PAIR_K
  FSIL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (c->timing) {  // the kernel alone, for the roofline (ms_score_kernel)
    FSIL_CUDA(cudaEventRecord(c->ev[7], c->stream));
    c->ev7_recorded = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = c->pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  static const bool prof = std::getenv("FSIL_TC_PROFILE") != nullptr;
  unsigned long long* dbg = nullptr;
  if (prof) {
    FSIL_CUDA(cudaMalloc(&dbg, 16 * sizeof(unsigned long long)));
    FSIL_CUDA(cudaMemsetAsync(dbg, 0, 16 * sizeof(unsigned long long), c->stream));
    if (std::atoi(std::getenv("FSIL_TC_PROFILE")) == 2) FSIL_CUDA(cudaMemsetAsync(dbg + 15, 1, 1, c->stream));
  }
  tp.dbg = dbg;
  FSIL_CUDA(cudaLaunchKernelEx(&cfg, kern, mx, mh, ml, mscr, mscst, tp, ntiles, ns, nb, nx));
  FSIL_LAUNCHED(c);
  if (dbg) {
    unsigned long long h[16];
    FSIL_CUDA(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    const char* names[15] = {"mma acc_empty", "mma a_full", "mma b_full", "mma total", "A stg_empty",
                             "A scr_ready", "B b_empty", "epi acc_full", "epi meta_full", "conv xs_full",
                             "(unused)", "mma issue", "mma items", "mma cbs", "conv scr_free"};
    const double pairs = static_cast<double>(grid / 2), ctas = static_cast<double>(grid);
    std::fprintf(stderr, "[fsil tc pair profile] ns=%d nb=%d nx=%d Mcycles per CTA (MMA rows: per pair):", ns, nb, nx);
    for (int i = 0; i < 15; ++i)
      std::fprintf(stderr, " %s=%.3f", names[i], h[i] / ((i < 4 || (i >= 10 && i < 14)) ? pairs : ctas) / 1e6);
    std::fprintf(stderr, "\n");
    cudaFree(dbg);
  }
}

}  // namespace tc
}  // namespace fsil
