// pipe_probe.cu -- microbenchmark of the per-SM throughput of the instructions the
// aggregation pass leans on (F2F.F64.F32 conversions, DFMA, DADD), on one B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void probe(const float* in, double* out, int iters) {
  float f0 = in[threadIdx.x & 31], f1 = f0 * 1.1f, f2 = f0 * 1.2f, f3 = f0 * 1.3f;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0) {  // conversions only (independent)
        a0 += (double)f0; a1 += (double)f1; a2 += (double)f2; a3 += (double)f3;
        f0 += 1.0f; f1 += 1.0f; f2 += 1.0f; f3 += 1.0f;
      } else if (MODE == 1) {  // dfma only
        a0 = fma(a0, 1.0000001, 0.5); a1 = fma(a1, 1.0000001, 0.5); a2 = fma(a2, 1.0000001, 0.5); a3 = fma(a3, 1.0000001, 0.5);
      } else {  // fp32 adds only (reference)
        f0 += 1.0f; f1 += 1.0f; f2 += 1.0f; f3 += 1.0f;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + f0 + f1 + f2 + f3;
}

int main() {
  float* in; double* out;
  cudaMalloc(&in, 128); cudaMalloc(&out, 148 * 4 * 1024 * 8);
  cudaMemset(in, 0, 128);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, blocks = 148 * 4, threads = 512;
  const char* names[3] = {"F2F.F64.F32 + DADD + FADD", "DFMA", "FADD"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) probe<0><<<blocks, threads>>>(in, out, iters);
      if (mode == 1) probe<1><<<blocks, threads>>>(in, out, iters);
      if (mode == 2) probe<2><<<blocks, threads>>>(in, out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double ops = double(blocks) * threads * iters * 8 * 4;  // per op type
      if (rep) printf("%-28s %.3f ms  %.1f Gop/s  = %.1f per SM per clk (at 1.965 GHz)\n", names[mode], ms,
                      ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
