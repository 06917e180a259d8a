// tc_probe.cu -- TEST INFRASTRUCTURE: the tcgen05 accumulation model the scoring
// pass's neighbour certificate charges (score_tc.cu, kMmaUlp), measured on the device.
//
// One CTA runs a 128 x N x (16 * ksteps) kind::f16 MMA chain exactly as the scoring
// kernel issues it (fp16 operands in the K-major SWIZZLE_128B layout, fp32 accumulator
// in TMEM, one tcgen05.mma per 16-element K step) and reads the accumulator back after
// EVERY step, so the host can compare each step against the exact sum of the previous
// accumulator and the step's 16 exact fp16 products (tests/test_tc_numerics.py).
// Not part of libfsil: built into libfsil_probe.so and loaded only by the tests.
#include <cuda_fp16.h>
#include <stdint.h>

#include "sm100.cuh"

namespace {

using namespace fsil::sm100;

constexpr int kM = 128;
constexpr int kN = 32;
constexpr int kMaxChunks = 4;  // K <= 256 (16 steps)

__global__ void __launch_bounds__(128, 1)
    tc_probe_kernel(const __half* __restrict__ A, const __half* __restrict__ B, int ksteps, float* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int nchunks = (ksteps + 3) / 4;
  uint8_t* sa = base;                           // [nchunks][128 rows x 128 B]
  uint8_t* sb = sa + nchunks * kM * 128;        // [nchunks][32 rows x 128 B]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + nchunks * kN * 128);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int K = 64 * nchunks;
  // operands -> the UMMA K-major SWIZZLE_128B layout (the converters' layout in score_tc)
  for (int e = threadIdx.x; e < kM * K; e += blockDim.x) {
    const int r = e / K, k = e % K, ch = k / 64, kk = k % 64;
    *reinterpret_cast<__half*>(sa + ch * kM * 128 + r * 128 + ((((kk >> 3) ^ (r & 7)) << 4)) + (kk & 7) * 2) =
        k < 16 * ksteps ? A[static_cast<int64_t>(r) * 16 * ksteps + k] : __float2half(0.f);
  }
  for (int e = threadIdx.x; e < kN * K; e += blockDim.x) {
    const int r = e / K, k = e % K, ch = k / 64, kk = k % 64;
    *reinterpret_cast<__half*>(sb + ch * kN * 128 + r * 128 + ((((kk >> 3) ^ (r & 7)) << 4)) + (kk & 7) * 2) =
        k < 16 * ksteps ? B[static_cast<int64_t>(r) * 16 * ksteps + k] : __float2half(0.f);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<32>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  constexpr uint32_t idesc = idesc_f16_f32(kM, kN);
  for (int s = 0; s < ksteps; ++s) {
    if (threadIdx.x == 0) {
      tc_fence_after();
      const int ch = s / 4, ks = s % 4;
      const uint64_t da = desc_k_sw128(smem_u32(sa + ch * kM * 128)) + 2 * ks;
      const uint64_t db = desc_k_sw128(smem_u32(sb + ch * kN * 128)) + 2 * ks;
      mma_f16(tmem, da, db, idesc, s > 0 ? 1u : 0u);
      mma_commit(bar);
    }
    mbar_wait(bar, s & 1);
    tc_fence_after();
    uint32_t v[32];
    tmem_ld32_issue(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
    tmem_ld_wait(v);
    const int row = warp * 32 + lane;
#pragma unroll
    for (int j = 0; j < 32; ++j) out[(static_cast<int64_t>(s) * kM + row) * kN + j] = __uint_as_float(v[j]);
    tc_fence_before();
    __syncthreads();
  }
  if (warp == 0) tmem_dealloc<32>(tmem);
}

}  // namespace

// A [128][16*ksteps], B [32][16*ksteps] fp16 row-major (host); out [ksteps][128][32] fp32
// (host): the accumulator after every K step.  Returns 0 or a CUDA error code.
extern "C" int fsil_tc_probe(const uint16_t* A, const uint16_t* B, int ksteps, float* out) {
  if (ksteps < 1 || ksteps > 4 * kMaxChunks) return -1;
  const size_t na = static_cast<size_t>(kM) * 16 * ksteps, nb = static_cast<size_t>(kN) * 16 * ksteps;
  const size_t no = static_cast<size_t>(ksteps) * kM * kN;
  __half *dA = nullptr, *dB = nullptr;
  float* dO = nullptr;
  cudaError_t e = cudaMalloc(&dA, na * 2);
  if (!e) e = cudaMalloc(&dB, nb * 2);
  if (!e) e = cudaMalloc(&dO, no * 4);
  if (!e) e = cudaMemcpy(dA, A, na * 2, cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(dB, B, nb * 2, cudaMemcpyHostToDevice);
  const int nchunks = (ksteps + 3) / 4;
  const int smem = 1024 + nchunks * (kM + kN) * 128 + 64;
  if (!e) e = cudaFuncSetAttribute(tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (!e) {
    tc_probe_kernel<<<1, 128, smem>>>(dA, dB, ksteps, dO);
    e = cudaGetLastError();
  }
  if (!e) e = cudaDeviceSynchronize();
  if (!e) e = cudaMemcpy(out, dO, no * 4, cudaMemcpyDeviceToHost);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
  return static_cast<int>(e);
}
