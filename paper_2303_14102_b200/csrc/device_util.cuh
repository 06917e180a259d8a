// device_util.cuh -- small sm_100a device helpers shared by the libfsil kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fsil {

// Programmatic dependent launch: wait until the stream predecessor grid has completed
// and its writes are visible (a no-op when the kernel was launched without PDL).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// Raw int32 label -> non-zero 64-bit hash-table key (0 marks an empty slot).
__device__ __forceinline__ unsigned long long label_key(int32_t lab) {
  return (1ull << 32) | static_cast<uint32_t>(lab);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int src_size = valid ? 16 : 0;  // 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_size));
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int src_size = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_size));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Streaming 128-bit global load that does not allocate in L1.
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void atomic_min_i64(int64_t* addr, int64_t v) {
  atomicMin(reinterpret_cast<long long*>(addr), static_cast<long long>(v));
}

// Max over non-negative floats via their ordered integer bit patterns.
__device__ __forceinline__ void atomic_max_nonneg_f32(float* addr, float v) {
  atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
}

// assemble_score + singleton convention (report.cpp:7-30).  a, b >= 0 after
// clamping, so the reference's negative-input throw cannot trigger.
__device__ __forceinline__ double assemble_score(double a, double b) {
  if (a == 0.0 && b == 0.0) return 0.0;
  return a <= b ? 1.0 - a / b : b / a - 1.0;
}

// Grid-wide barrier for a co-resident (cooperatively launched) grid: arrival count
// plus a generation word; the last arriver resets the count and bumps the generation.
__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = gen;
    const unsigned int g0 = *vgen;
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0u;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vgen == g0) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

}  // namespace fsil
