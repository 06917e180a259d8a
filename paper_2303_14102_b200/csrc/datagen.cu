// datagen.cu -- synthetic inputs for the five BASELINE.json configurations.
//
// Not on the measured path: it creates the seeded inputs that the benchmark
// and the parity tests feed, identically, to libfsil and to the CPU oracle.
//
//   C1  fsilgen_blobs_host: the reference's own generator, restated
//       (blobs.hpp:13-44, blobs.cpp:11-54): SplitMix64 + Box-Muller, centres
//       first, then points in dataset order, label i mod k; fp64, rounded to fp32.
//   C2..C5 fsilgen_device: counter-based SplitMix64 normals (each value is a
//       pure function of (seed, stream, index), so any row range can be
//       regenerated), one warp per point, fp32 Box-Muller.
//         2: cosine directions ~ N(0,I) normalised; x = normalise(dir + 0.1 N)
//            * U(0.5, 5); labels i.i.d. uniform
//         3: centres 5 N(0,I); x = centre + N; Zipf(1.1) sizes (smallest two
//            forced to 1 and 2), labels shuffled
//         4: centres 3 N(0,I); x = uniformly chosen centre + N; label =
//            nearest centre (fp64, lowest index on ties)
//         5: directions uniform on the sphere; x = normalise(dir + 0.3 N) *
//            LogNormal(0, 0.25); Dirichlet(0.5) sizes with floor 1, shuffled
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// i-th SplitMix64 output (0-based) of a generator seeded with `seed`.
__host__ __device__ inline uint64_t splitmix_at(uint64_t seed, uint64_t i) {
  return mix64(seed + (i + 1) * kGolden);
}
__host__ __device__ inline uint64_t stream_seed(uint64_t seed, uint64_t stream) {
  return mix64(seed ^ (stream * 0xD1B54A32D192ED03ULL));
}
__device__ inline float unit_f(uint64_t u) { return static_cast<float>(u >> 40) * 0x1.0p-24f; }
// Standard normal #j of a stream: uniforms 2m, 2m+1 with m = j/2 (Box-Muller).
__device__ inline float normal_f(uint64_t seed, uint64_t j) {
  const uint64_t m = j >> 1;
  const float u1 = unit_f(splitmix_at(seed, 2 * m));
  const float u2 = unit_f(splitmix_at(seed, 2 * m + 1));
  const float r = sqrtf(-2.0f * log1pf(-u1));
  float s, c;
  sincospif(2.0f * u2, &s, &c);
  return (j & 1) ? r * s : r * c;
}

// ---------------------------------------------------------------- C1 (host) --
struct SplitMix64 {  // blobs.hpp:13-30
  uint64_t state;
  uint64_t next_u64() {
    state += kGolden;
    return mix64(state);
  }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
};
struct GaussianStream {  // blobs.cpp:11-23
  SplitMix64 rng;
  double spare = 0.0;
  bool has_spare = false;
  double next() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = rng.next_unit(), u2 = rng.next_unit();
    const double r = std::sqrt(-2.0 * std::log1p(-u1));
    const double theta = 2.0 * M_PI * u2;
    spare = r * std::sin(theta);
    has_spare = true;
    return r * std::cos(theta);
  }
};

// ---------------------------------------------------------------- kernels ----
__global__ void centres_kernel(uint64_t seed, int k, int d, float scale, bool normalise,
                               double* centres) {
  const int c = blockIdx.x;
  __shared__ double red[32];
  double ss = 0.0;
  for (int l = threadIdx.x; l < d; l += blockDim.x) {
    const double v = scale * normal_f(seed, static_cast<uint64_t>(c) * d + l);
    centres[static_cast<int64_t>(c) * d + l] = v;
    ss += v * v;
  }
  if (!normalise) return;
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) t += red[w];
    red[0] = sqrt(t);
  }
  __syncthreads();
  for (int l = threadIdx.x; l < d; l += blockDim.x) centres[static_cast<int64_t>(c) * d + l] /= red[0];
}

__global__ void uniform_labels_kernel(uint64_t seed, int64_t row0, int64_t n, int k, int32_t* labels) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t u = splitmix_at(seed, row0 + i);
  labels[i] = static_cast<int32_t>((u >> 32) * static_cast<uint64_t>(k) >> 32);
}

// One warp per point.  mode: 0 = centre + sigma N (sqeuclid), 1 = normalise(dir +
// sigma N) * magnitude (cosine; mag_kind 0: U(0.5,5), 1: LogNormal(0, 0.25)).  Local row i
// is global row row0 + i: every value is a function of the global index.
__global__ void points_kernel(uint64_t seed_noise, uint64_t seed_mag, int64_t row0, int64_t n, int d,
                              const double* centres, const int32_t* labels, float sigma, int mode,
                              int mag_kind, float* X) {
  const int64_t li = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (li >= n) return;
  const int64_t i = row0 + li;
  const int lab = labels[li];
  const double* c = centres + static_cast<int64_t>(lab) * d;
  float* x = X + li * d;
  if (mode == 0) {
    for (int l = lane; l < d; l += 32)
      x[l] = static_cast<float>(c[l] + sigma * normal_f(seed_noise, static_cast<uint64_t>(i) * d + l));
    return;
  }
  float ss = 0.f;
  for (int l = lane; l < d; l += 32) {
    const float v = static_cast<float>(c[l]) + sigma * normal_f(seed_noise, static_cast<uint64_t>(i) * d + l);
    x[l] = v;
    ss += v * v;
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  float mag;
  if (mag_kind == 0) mag = 0.5f + 4.5f * unit_f(splitmix_at(seed_mag, i));
  else mag = expf(0.25f * normal_f(seed_mag, static_cast<uint64_t>(i)));
  const float scale = mag / sqrtf(ss);
  __syncwarp();
  for (int l = lane; l < d; l += 32) x[l] *= scale;
}

// C4: label = nearest centre of the stored fp32 point (fp64, lowest index on ties).
__global__ void nearest_kernel(const float* X, int64_t n, int d, const double* __restrict__ cs,
                               int k, int32_t* labels) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* x = X + i * d;
  double best = INFINITY;
  int arg = 0;
  for (int c = 0; c < k; ++c) {
    double acc = 0.0;
    for (int l = 0; l < d; ++l) {
      const double t = static_cast<double>(x[l]) - cs[c * d + l];
      acc = fma(t, t, acc);
    }
    if (acc < best) {
      best = acc;
      arg = c;
    }
  }
  labels[i] = arg;
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

double host_unit(uint64_t seed, uint64_t i) {
  return static_cast<double>(splitmix_at(seed, i) >> 11) * 0x1.0p-53;
}

// Largest-remainder integer sizes summing to n with a floor of `floor1` per cluster.
std::vector<int64_t> apportion(const std::vector<double>& p, int64_t n, int64_t floor1) {
  const size_t k = p.size();
  const double tot = std::accumulate(p.begin(), p.end(), 0.0);
  std::vector<int64_t> sz(k);
  std::vector<std::pair<double, size_t>> rem(k);
  int64_t used = 0;
  for (size_t j = 0; j < k; ++j) {
    const double q = p[j] / tot * static_cast<double>(n);
    sz[j] = static_cast<int64_t>(std::floor(q));
    rem[j] = {q - static_cast<double>(sz[j]), j};
    used += sz[j];
  }
  std::sort(rem.begin(), rem.end(), [](auto& a, auto& b) {
    return a.first != b.first ? a.first > b.first : a.second < b.second;
  });
  for (int64_t r = 0; r < n - used; ++r) sz[rem[static_cast<size_t>(r) % k].second] += 1;
  for (size_t j = 0; j < k; ++j) {
    while (sz[j] < floor1) {  // take from the largest cluster
      const size_t big = static_cast<size_t>(std::max_element(sz.begin(), sz.end()) - sz.begin());
      sz[big] -= 1;
      sz[j] += 1;
    }
  }
  return sz;
}

std::vector<int32_t> shuffled_labels(const std::vector<int64_t>& sizes, uint64_t seed) {
  int64_t n = std::accumulate(sizes.begin(), sizes.end(), int64_t(0));
  std::vector<int32_t> lab(static_cast<size_t>(n));
  int64_t pos = 0;
  for (size_t j = 0; j < sizes.size(); ++j)
    for (int64_t t = 0; t < sizes[j]; ++t) lab[pos++] = static_cast<int32_t>(j);
  SplitMix64 rng{seed};
  for (int64_t i = n - 1; i > 0; --i) {  // Fisher-Yates
    const uint64_t r = rng.next_u64();
    const int64_t j = static_cast<int64_t>((static_cast<unsigned __int128>(r) * (i + 1)) >> 64);
    std::swap(lab[i], lab[j]);
  }
  return lab;
}

double gamma_variate(double shape, SplitMix64& rng, GaussianStream& g) {
  // Marsaglia-Tsang for shape >= 1; boost for shape < 1.
  double boost = 1.0;
  if (shape < 1.0) {
    boost = std::pow(rng.next_unit() + 1e-300, 1.0 / shape);
    shape += 1.0;
  }
  const double dd = shape - 1.0 / 3.0, cc = 1.0 / std::sqrt(9.0 * dd);
  for (;;) {
    double x, v;
    do {
      x = g.next();
      v = 1.0 + cc * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = rng.next_unit();
    if (u < 1.0 - 0.0331 * x * x * x * x) return dd * v * boost;
    if (std::log(u) < 0.5 * x * x + dd * (1.0 - v + std::log(v))) return dd * v * boost;
  }
}

}  // namespace

extern "C" {

// C1: the reference blob generator (blobs.cpp:25-54) restated on the host.
int fsilgen_blobs_host(int64_t n, int32_t d, int32_t k, double spread, double separation,
                       uint64_t seed, float* X, int32_t* labels) {
  if (k < 2 || n < k || d < 1 || !(spread > 0.0)) return 2;
  GaussianStream normals{SplitMix64{seed}};
  std::vector<double> centres(static_cast<size_t>(k) * d);
  for (int32_t c = 0; c < k; ++c)
    for (int32_t l = 0; l < d; ++l) centres[static_cast<size_t>(c) * d + l] = separation * normals.next();
  for (int64_t i = 0; i < n; ++i) {
    const int32_t c = static_cast<int32_t>(i % k);
    labels[i] = c;
    for (int32_t l = 0; l < d; ++l)
      X[i * d + l] = static_cast<float>(centres[static_cast<size_t>(c) * d + l] + spread * normals.next());
  }
  return 0;
}

// C2..C5 on the device, rows [row0, row0 + n) of the n_global-row dataset (any rank's
// shard of one global dataset: the same bytes as rows row0.. of the whole).  Returns 0 on
// success; dX [n*d] fp32, dlabels [n].
int fsilgen_device_rows(int config, int64_t n_global, int64_t row0, int64_t n, int32_t d, int32_t k,
                        uint64_t seed, float* dX, int32_t* dlabels, void* stream_ptr, char* err, size_t errlen) {
  cudaStream_t st = static_cast<cudaStream_t>(stream_ptr);
  try {
    if (n_global < 2 || d < 1 || k < 2 || row0 < 0 || n < 1 || row0 + n > n_global)
      throw std::runtime_error("bad generator shape");
    double* centres = nullptr;
    check(cudaMalloc(&centres, static_cast<size_t>(k) * d * sizeof(double)), "cudaMalloc");
    const uint64_t s_cent = stream_seed(seed, 1), s_noise = stream_seed(seed, 2),
                   s_lab = stream_seed(seed, 3), s_mag = stream_seed(seed, 4),
                   s_shuf = stream_seed(seed, 5), s_size = stream_seed(seed, 6);
    const unsigned warps_grid = static_cast<unsigned>((n * 32 + 255) / 256);
    const unsigned thr_grid = static_cast<unsigned>((n + 255) / 256);
    switch (config) {
      case 2: {
        centres_kernel<<<k, 128, 0, st>>>(s_cent, k, d, 1.0f, true, centres);
        uniform_labels_kernel<<<thr_grid, 256, 0, st>>>(s_lab, row0, n, k, dlabels);
        points_kernel<<<warps_grid, 256, 0, st>>>(s_noise, s_mag, row0, n, d, centres, dlabels, 0.1f, 1, 0, dX);
        break;
      }
      case 3: {
        std::vector<double> p(static_cast<size_t>(k));
        for (int32_t j = 0; j < k; ++j) p[j] = std::pow(static_cast<double>(j + 1), -1.1);
        auto sz = apportion(p, n_global, 1);
        // force the two smallest clusters to sizes 1 and 2 (singleton path)
        std::vector<size_t> idx(static_cast<size_t>(k));
        std::iota(idx.begin(), idx.end(), 0);
        std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return sz[a] < sz[b]; });
        const int64_t give = (sz[idx[0]] - 1) + (sz[idx[1]] - 2);
        sz[idx[0]] = 1;
        sz[idx[1]] = 2;
        sz[idx.back()] += give;
        auto lab = shuffled_labels(sz, s_shuf);
        check(cudaMemcpyAsync(dlabels, lab.data() + row0, n * sizeof(int32_t), cudaMemcpyHostToDevice, st), "H2D");
        centres_kernel<<<k, 128, 0, st>>>(s_cent, k, d, 5.0f, false, centres);
        points_kernel<<<warps_grid, 256, 0, st>>>(s_noise, s_mag, row0, n, d, centres, dlabels, 1.0f, 0, 0, dX);
        check(cudaStreamSynchronize(st), "sync");
        break;
      }
      case 4: {
        centres_kernel<<<k, 128, 0, st>>>(s_cent, k, d, 3.0f, false, centres);
        uniform_labels_kernel<<<thr_grid, 256, 0, st>>>(s_lab, row0, n, k, dlabels);
        points_kernel<<<warps_grid, 256, 0, st>>>(s_noise, s_mag, row0, n, d, centres, dlabels, 1.0f, 0, 0, dX);
        nearest_kernel<<<thr_grid, 256, 0, st>>>(dX, n, d, centres, k, dlabels);
        break;
      }
      case 5: {
        SplitMix64 rng{s_size};
        GaussianStream g{SplitMix64{s_size ^ 0x5555}};
        std::vector<double> p(static_cast<size_t>(k));
        for (auto& v : p) v = gamma_variate(0.5, rng, g);
        auto sz = apportion(p, n_global, 1);
        auto lab = shuffled_labels(sz, s_shuf);
        check(cudaMemcpyAsync(dlabels, lab.data() + row0, n * sizeof(int32_t), cudaMemcpyHostToDevice, st), "H2D");
        centres_kernel<<<k, 128, 0, st>>>(s_cent, k, d, 1.0f, true, centres);
        points_kernel<<<warps_grid, 256, 0, st>>>(s_noise, s_mag, row0, n, d, centres, dlabels, 0.3f, 1, 1, dX);
        check(cudaStreamSynchronize(st), "sync");
        break;
      }
      default:
        throw std::runtime_error("unknown generator config " + std::to_string(config));
    }
    check(cudaGetLastError(), "generator launch");
    check(cudaStreamSynchronize(st), "generator sync");
    cudaFree(centres);
    return 0;
  } catch (const std::exception& e) {
    if (err && errlen) {
      snprintf(err, errlen, "%s", e.what());
    }
    return 1;
  }
}

int fsilgen_device(int config, int64_t n, int32_t d, int32_t k, uint64_t seed, float* dX, int32_t* dlabels,
                   void* stream_ptr, char* err, size_t errlen) {
  return fsilgen_device_rows(config, n, 0, n, d, k, seed, dX, dlabels, stream_ptr, err, errlen);
}

}  // extern "C"
