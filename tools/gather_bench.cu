// Builder probe (not product code): HBM throughput of gathering whole fp32 rows (D = 768,
// 3 KB) in a random order, the access pattern of the label-sorted aggregation and of a
// cluster-ordered exact pass, against streaming the same rows in order.
//   (a) cp.async.bulk ring: W warps per CTA, R one-row slots per warp (the aggregation's scheme)
//   (b) plain 16-byte vector loads: each warp loads U rows at once (U x 6 float4 per lane)
// Each row is consumed by a light fp32 sum so no load is dead.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2303_14102_b200/csrc tools/gather_bench.cu -o tools/gather_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace fsil::sm100;

constexpr int D = 768, ROWB = D * 4;

__global__ void __launch_bounds__(256, 1) ring_kernel(const float* __restrict__ X, const int* __restrict__ order,
                                                      int64_t n, int R, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint8_t* ring = sm + static_cast<size_t>(w) * R * ROWB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(nw) * R * ROWB) + w * R;
  if (lane == 0)
    for (int s = 0; s < R; ++s) mbar_init(bars + s, 1);
  fence_barrier_init();
  __syncwarp();
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * nw + w, nwarps = static_cast<int64_t>(gridDim.x) * nw;
  const int64_t per = (n + nwarps - 1) / nwarps, b0 = gw * per, b1 = min(n, b0 + per);
  const int64_t iters = b1 > b0 ? b1 - b0 : 0;
  auto fill = [&](int64_t it, int s) {
    if (lane == 0) {
      mbar_arrive_expect_tx(bars + s, ROWB);
      bulk_load(ring + static_cast<size_t>(s) * ROWB, X + static_cast<int64_t>(order[b0 + it]) * D, ROWB, bars + s);
    }
  };
  for (int j = 0; j < R && j < iters; ++j) fill(j, j);
  float acc = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t it = 0; it < iters; ++it) {
    mbar_wait(bars + s, ph);
    const float4* row = reinterpret_cast<const float4*>(ring + static_cast<size_t>(s) * ROWB);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const float4 t = row[lane + 32 * q];
      acc += (t.x + t.y) + (t.z + t.w);
    }
    __syncwarp();
    if (it + R < iters) fill(it + R, s);
    if (++s == R) {
      s = 0;
      ph ^= 1u;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) load_kernel(const float* __restrict__ X, const int* __restrict__ order,
                                                   int64_t n, float* out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * nw + w, nwarps = static_cast<int64_t>(gridDim.x) * nw;
  float acc = 0.f;
  for (int64_t b = gw * U; b < n; b += nwarps * U) {
    float4 t[U][6];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = b + u < n ? b + u : n - 1;
      const float4* row = reinterpret_cast<const float4*>(X + static_cast<int64_t>(order[i]) * D);
#pragma unroll
      for (int q = 0; q < 6; ++q) t[u][q] = __ldg(row + lane + 32 * q);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < 6; ++q) acc += (t[u][q].x + t[u][q].y) + (t[u][q].z + t[u][q].w);
  }
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 8000000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* X;
  int *ord_rand, *ord_seq;
  float* out;
  cudaMalloc(&X, n * ROWB);
  cudaMemset(X, 0, n * ROWB);
  cudaMalloc(&ord_rand, n * 4);
  cudaMalloc(&ord_seq, n * 4);
  cudaMalloc(&out, 4);
  std::vector<int> h(n);
  for (int64_t i = 0; i < n; ++i) h[i] = static_cast<int>(i);
  cudaMemcpy(ord_seq, h.data(), n * 4, cudaMemcpyHostToDevice);
  srand(7);
  for (int64_t i = n - 1; i > 0; --i) {
    const int64_t j = (static_cast<int64_t>(rand()) * RAND_MAX + rand()) % (i + 1);
    std::swap(h[i], h[j]);
  }
  cudaMemcpy(ord_rand, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    std::printf("%-34s %8.3f ms  %7.0f GB/s  err=%s\n", name, best, n * double(ROWB) / (best * 1e6),
                cudaGetErrorString(cudaGetLastError()));
  };
  for (int rnd = 0; rnd < 2; ++rnd) {
    const int* ord = rnd ? ord_rand : ord_seq;
    const char* tag = rnd ? "random" : "sequential";
    for (int W : {8, 16}) {
      for (int R : {2, 4, 8, 12}) {
        const size_t smem = static_cast<size_t>(W) * R * (ROWB + 8);
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        char name[96];
        std::snprintf(name, sizeof name, "%s ring W=%d R=%d", tag, W, R);
        timeit(name, [&] { ring_kernel<<<sms, W * 32, smem>>>(X, ord, n, R, out); });
      }
    }
    char name[96];
    std::snprintf(name, sizeof name, "%s loads U=2", tag);
    timeit(name, [&] { load_kernel<2><<<sms * 8, 256>>>(X, ord, n, out); });
    std::snprintf(name, sizeof name, "%s loads U=4", tag);
    timeit(name, [&] { load_kernel<4><<<sms * 8, 256>>>(X, ord, n, out); });
    std::snprintf(name, sizeof name, "%s loads U=4 (4 CTA/SM)", tag);
    timeit(name, [&] { load_kernel<4><<<sms * 4, 256>>>(X, ord, n, out); });
  }
  return 0;
}
