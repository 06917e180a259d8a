// Builder probe (not product code): tensor-core issue rate of tcgen05.mma kind::f16 (K = 16)
// against kind::i8 (K = 32) for a 128 x 256 tile with operands resident in shared memory,
// one CTA per SM, every SM busy.  Prints cycles per MMA and dense ops per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2303_14102_b200/csrc tools/mma_rate.cu -o tools/mma_rate
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fsil::sm100;

__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <bool I8>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    // A: 128 rows x 128 B (K-major SW128), B: 256 rows x 128 B
    const uint64_t da = desc_k_sw128(smem_u32(base)), db = desc_k_sw128(smem_u32(base + 16384));
    const uint32_t idesc = I8 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24))
                              : idesc_f16_f32(128, 256);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (i & 1) * 256;
      if (I8) mma_i8(d, da + 2 * (i & 3), db + 2 * (i & 3), idesc, 1u);
      else mma_f16(d, da + 2 * (i & 3), db + 2 * (i & 3), idesc, 1u);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* dc;
  cudaMalloc(&dc, sms * sizeof(long long));
  const int iters = 200000;
  for (int pass = 0; pass < 2; ++pass) {
    for (int i8 = 0; i8 < 2; ++i8) {
      auto k = i8 ? rate_kernel<true> : rate_kernel<false>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<sms, 128, 100 * 1024>>>(iters, dc);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      long long h[256];
      cudaMemcpy(h, dc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < sms; ++i) cyc += h[i];
      cyc /= sms;
      const double kdim = i8 ? 32 : 16;
      const double ops = 2.0 * 128 * 256 * kdim;
      std::printf("%s: err=%s  %.1f cycles/MMA  %.0f ops/clk/SM  %.1f ms  %.1f Tops/s (all SMs)\n",
                  i8 ? "kind::i8  128x256x32" : "kind::f16 128x256x16", cudaGetErrorString(err), cyc / iters,
                  ops / (cyc / iters), ms, ops * iters * sms / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
