// stream_probe.cu -- what read bandwidth does one persistent CTA per SM reach when it
// streams a large array through an NS-stage ring of bulk copies (cp.async.bulk +
// mbarrier), against a plain many-warp LDG.128 reduction?  Sizes the scoring /
// aggregation pipelines' bytes in flight.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void marrive(uint64_t* b) {
  asm volatile("{.reg .b64 s; mbarrier.arrive.shared::cta.b64 s, [%0];}" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t n) {
  asm volatile("{.reg .b64 s; mbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;}" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph), "r"(0x989680) : "memory");
}

__global__ void ring(const uint8_t* X, size_t bytes, int stage, int ns, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)ns * stage);
  uint64_t* empty = full + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) { for (int i = 0; i < ns; ++i) { minit(full + i, 1); minit(empty + i, W); } }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const size_t nst = bytes / stage;
  if (warp == W) {
    if (lane == 0) {
      int i = 0;
      for (size_t s = blockIdx.x; s < nst; s += gridDim.x, ++i) {
        const int b = i % ns;
        mwait(empty + b, ((i / ns) & 1) ^ 1);
        mexpect(full + b, stage);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(sm + (size_t)b * stage)), "l"(X + s * stage), "r"(stage), "r"(su32(full + b)) : "memory");
      }
    }
    return;
  }
  float acc = 0.f;
  int i = 0;
  for (size_t s = blockIdx.x; s < nst; s += gridDim.x, ++i) {
    const int b = i % ns;
    mwait(full + b, (i / ns) & 1);
    acc += ((const float*)(sm + (size_t)b * stage))[threadIdx.x];  // touch one word per thread
    __syncwarp();
    if (lane == 0) marrive(empty + b);
  }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void ldg(const float4* X, size_t n4, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(X + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) out[0] = acc;
}


// the scoring kernel's staging: two 2-D tensor boxes (128 rows x 32 fp32, 128B swizzle)
// per 32 KB stage of a [N][64] fp32 matrix
__global__ void ring2d(const __grid_constant__ CUtensorMap tm, int64_t nrows, int ns, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  const int stage = 32768;
  uint64_t* full = (uint64_t*)(base + (size_t)ns * stage);
  uint64_t* empty = full + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) { for (int i = 0; i < ns; ++i) { minit(full + i, 1); minit(empty + i, W); } }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int64_t ntl = nrows / 128;
  if (warp == W) {
    if (lane == 0) {
      int i = 0;
      for (int64_t t = blockIdx.x; t < ntl; t += gridDim.x, ++i) {
        const int b = i % ns;
        mwait(empty + b, ((i / ns) & 1) ^ 1);
        mexpect(full + b, stage);
        for (int bx = 0; bx < 2; ++bx)
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(su32(base + (size_t)b * stage + bx * 16384)), "l"((uint64_t)&tm), "r"(bx * 32), "r"((int)(t * 128)),
                       "r"(su32(full + b)) : "memory");
      }
    }
    return;
  }
  float acc = 0.f;
  int i = 0;
  for (int64_t t = blockIdx.x; t < ntl; t += gridDim.x, ++i) {
    const int b = i % ns;
    mwait(full + b, (i / ns) & 1);
    acc += ((const float*)(base + (size_t)b * stage))[threadIdx.x];
    __syncwarp();
    if (lane == 0) marrive(empty + b);
  }
  if (acc == 1234.5f) out[0] = acc;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t bytes = 256ull << 20;
  uint8_t* X; float* out;
  cudaMalloc(&X, bytes + (1 << 20)); cudaMalloc(&out, 64);
  cudaMemset(X, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  auto t = [&](auto f) { f(); cudaEventRecord(e0); for (int r = 0; r < 5; ++r) f(); cudaEventRecord(e1);
                         cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 5; };
  float ms = t([&] { ldg<<<sms * 8, 512>>>((const float4*)X, bytes / 16, out); });
  printf("LDG.128 many warps: %.1f us  %.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
  for (int stage : {8192, 16384, 32768, 65536})
    for (int ns : {2, 3, 4, 6}) {
      if ((size_t)stage * ns > 200 * 1024) continue;
      for (int warps : {4, 8}) {
        ms = t([&] { ring<<<sms, (warps + 1) * 32, stage * ns + 256>>>(X, bytes, stage, ns, out); });
        printf("bulk ring stage %5d x %d, %d consumer warps: %.1f us  %.0f GB/s  (%.0f KB in flight/SM)\n", stage, ns,
               warps, ms * 1e3, bytes / ms / 1e6, stage * ns / 1024.0);
      }
    }
  {
    void* fp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncFn enc = (EncFn)fp;
    const int64_t nrows = bytes / 256;
    for (int prom = 0; prom < 2; ++prom) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {64, (cuuint64_t)nrows}, str[1] = {256};
      cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cudaFuncSetAttribute(ring2d, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      for (int ns : {2, 3, 4, 5, 6}) {
        ms = t([&] { ring2d<<<sms, 5 * 32, 32768 * ns + 1024 + 256>>>(tm, nrows, ns, out); });
        printf("tensor 2x(128x32 fp32 SW128) ring x %d, L2 promo %s: %.1f us  %.0f GB/s\n", ns, prom ? "256B" : "none",
               ms * 1e3, bytes / ms / 1e6);
      }
    }
  }
  return 0;
}
