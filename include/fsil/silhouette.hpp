// fsil/silhouette.hpp -- C++ host interface of the B200 Silhouette library, mirroring the
// reference fastsil library's public entry point so a caller switches by changing the
// namespace and handing over fp32 or fp64 features:
//
//   reference (/root/reference/proj/include/fastsil)          here (header-only, over fsil.h)
//   ---------------------------------------------------------  ---------------------------------
//   enum class Metric / Engine            types.hpp:20-30       fsil::Metric / fsil::Engine
//   metric_name / engine_name / parse_*   types.hpp:32-38       same names
//   ValidationError / IoError             types.hpp:41-50       same names (+ CudaError)
//   PointScore                            report.hpp:10-16      same fields, same order
//   SilhouetteReport                      report.hpp:18-26      same fields
//   assemble_score                        report.hpp:30         fsil::assemble_score
//   ShardPlan / plan_shards               engine.hpp:20-26      fsil::ShardPlan / plan_shards
//   compute_silhouette(Dataset, Metric, Engine, shards)
//                                         engine.hpp:124-125    compute_silhouette(X, labels, ...)
//
// The reference's Dataset (an Eigen D x N fp64 matrix + densified labels) is replaced by
// the raw inputs of validate_and_densify (dataset.hpp:46-48): an N x D row-major fp32 or
// fp64 matrix -- byte-compatible with a column-major D x N one -- and raw int labels.  The
// same validation runs on the device, in the reference's order, and fails with the
// same exception types.  Engine::Naive runs the Theta(N^2 D) engine (naive.cpp) on the
// GPU in fp64 -- the only engine for Metric::Euclidean.
#pragma once

#include <chrono>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <type_traits>
#include <utility>
#include <vector>

#include "fsil.h"

namespace fsil {

enum class Metric { SquaredEuclidean, Cosine, Euclidean };
enum class Engine { Fast, Naive };

inline std::string_view metric_name(Metric m) {
  switch (m) {
    case Metric::SquaredEuclidean: return "squared_euclidean";
    case Metric::Cosine: return "cosine";
    case Metric::Euclidean: return "euclidean_oracle";
  }
  return "unknown";
}
inline std::string_view engine_name(Engine e) { return e == Engine::Fast ? "fast" : "naive"; }
inline std::optional<Metric> parse_metric(std::string_view s) {
  if (s == "sqeuclid" || s == "squared_euclidean") return Metric::SquaredEuclidean;
  if (s == "cosine") return Metric::Cosine;
  if (s == "euclid" || s == "euclidean" || s == "euclidean_oracle") return Metric::Euclidean;
  return std::nullopt;
}
inline std::optional<Engine> parse_engine(std::string_view s) {
  if (s == "fast") return Engine::Fast;
  if (s == "naive") return Engine::Naive;
  return std::nullopt;
}

/// Input violated a dataset or argument invariant (reference CLI exit code 2).
class ValidationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
/// Filesystem-level failure (reference CLI exit code 1).
class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
/// No usable sm_100 device, or a CUDA / collective failure.  There is no CPU fallback.
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct PointScore {
  double a = 0.0;  // mean distance to the other members of the own cluster
  double b = 0.0;  // smallest mean distance to a foreign cluster
  double s = 0.0;  // silhouette, in [-1, 1]
  int own_cluster = -1;
  int neighbour_cluster = -1;
};

struct SilhouetteReport {
  std::vector<PointScore> scores;  // dataset order
  double mean = 0.0;
  Metric metric = Metric::SquaredEuclidean;
  Engine engine = Engine::Fast;
  int shards = 1;  // GPUs that scored the rows (the reference: host threads)
  double wall_time_ms = 0.0;
  std::vector<std::string> cluster_names;  // dense index -> original label
};

namespace detail {
inline void check(fsil_status st, const char* msg) {
  switch (st) {
    case FSIL_OK: return;
    case FSIL_ERR_VALIDATION: throw ValidationError(msg ? msg : "validation error");
    case FSIL_ERR_IO: throw IoError(msg ? msg : "io error");
    case FSIL_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg ? msg : "invalid argument");
    default: throw CudaError(msg ? msg : "device failure");
  }
}
inline int metric_code(Metric m) {
  return m == Metric::SquaredEuclidean ? FSIL_SQEUCLID : m == Metric::Cosine ? FSIL_COSINE : FSIL_EUCLID;
}
}  // namespace detail

/// (b - a) / max(a, b); 0 when both are 0; throws std::invalid_argument on negative input.
inline double assemble_score(double a, double b) {
  double s = 0.0;
  detail::check(fsil_assemble_score(a, b, &s), "assemble_score: negative mean distance");
  return s;
}

struct ShardPlan {
  std::vector<std::pair<int64_t, int64_t>> ranges;  // [begin, end) per shard
  int num_shards = 0;
};
/// min(requested, n) contiguous ranges; the first n mod w' take one extra row.
inline ShardPlan plan_shards(int64_t n, int requested) {
  std::vector<int64_t> buf(2 * static_cast<size_t>(requested > 0 ? requested : 1));
  int32_t w = 0;
  detail::check(fsil_plan_shards(n, requested, buf.data(), &w), "plan_shards: need n >= 1 and shards >= 1");
  ShardPlan p;
  p.num_shards = w;
  for (int i = 0; i < w; ++i) p.ranges.emplace_back(buf[2 * i], buf[2 * i + 1]);
  return p;
}

/// One device (CUDA ordinal), its stream and scratch.  Not shared by concurrent host threads.
class Context {
 public:
  explicit Context(int device = 0) {
    fsil_context* c = nullptr;
    const fsil_status st = fsil_create(&c, device);
    if (st != FSIL_OK) detail::check(st, fsil_last_error(nullptr));
    ctx_ = c;
  }
  ~Context() { fsil_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  Context(Context&& o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)) {}

  fsil_context* handle() const { return ctx_; }
  void set_stream(void* cuda_stream) { check(fsil_set_stream(ctx_, cuda_stream)); }
  void set_path(fsil_path p) { check(fsil_set_path(ctx_, p)); }
  void set_timing(bool on) { check(fsil_set_timing(ctx_, on ? 1 : 0)); }
  fsil_stats stats() const {
    fsil_stats s{};
    check(fsil_get_stats(ctx_, &s));
    return s;
  }
  void check(fsil_status st) const { detail::check(st, fsil_last_error(ctx_)); }

 private:
  fsil_context* ctx_ = nullptr;
};

namespace detail {
inline fsil_status call_host(fsil_context* c, int m, const float* X, const int32_t* L, int64_t n, int32_t d,
                             double* s, int32_t* nb, int32_t* own, double* a, double* b, double* mean,
                             int32_t* k, int32_t* raw) {
  return fsil_silhouette(c, m, X, L, n, d, s, nb, own, a, b, mean, k, raw);
}
inline fsil_status call_host(fsil_context* c, int m, const double* X, const int32_t* L, int64_t n, int32_t d,
                             double* s, int32_t* nb, int32_t* own, double* a, double* b, double* mean,
                             int32_t* k, int32_t* raw) {
  return fsil_silhouette_f64(c, m, X, L, n, d, s, nb, own, a, b, mean, k, raw);
}
}  // namespace detail

/// compute_silhouette(validate_and_densify(X, labels), metric, engine, shards)
/// (engine.hpp:124-125; dataset.hpp:48).  X: n x d row-major features in host memory,
/// fp32 or fp64 -- fp64 is the reference's own Matrix (Eigen::MatrixXd, D x N
/// column-major: pass .data()), aggregated and refined exactly in fp64; labels: n raw
/// ints.  `shards` is accepted for signature compatibility: the rows are scored by this
/// context's GPU (the multi-GPU path is the sharded protocol in fsil.h).
template <typename T>
inline SilhouetteReport compute_silhouette(Context& ctx, const T* X, const int32_t* labels, int64_t n,
                                           int32_t d, Metric metric, Engine engine = Engine::Fast,
                                           int shards = 0) {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "features are fp32 or fp64");
  (void)shards;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<double> s(static_cast<size_t>(n)), a(static_cast<size_t>(n)), b(static_cast<size_t>(n));
  std::vector<int32_t> nb(static_cast<size_t>(n)), own(static_cast<size_t>(n)), raw(static_cast<size_t>(n));
  double mean = 0.0;
  int32_t k = 0;
  if (engine == Engine::Naive) {  // the Theta(N^2 D) engine (fp64 features; fsil_silhouette_naive)
    std::vector<double> x64;
    const double* xp = nullptr;
    if constexpr (std::is_same_v<T, double>) {
      xp = X;
    } else {
      x64.assign(X, X + static_cast<size_t>(n) * static_cast<size_t>(d));
      xp = x64.data();
    }
    ctx.check(fsil_silhouette_naive(ctx.handle(), detail::metric_code(metric), xp, labels, n, d, s.data(), nb.data(),
                                    own.data(), a.data(), b.data(), &mean, &k, raw.data()));
  } else {
    ctx.check(detail::call_host(ctx.handle(), detail::metric_code(metric), X, labels, n, d, s.data(), nb.data(),
                                own.data(), a.data(), b.data(), &mean, &k, raw.data()));
  }
  SilhouetteReport r;
  r.scores.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    PointScore& p = r.scores[static_cast<size_t>(i)];
    p.a = a[static_cast<size_t>(i)];
    p.b = b[static_cast<size_t>(i)];
    p.s = s[static_cast<size_t>(i)];
    p.own_cluster = own[static_cast<size_t>(i)];
    p.neighbour_cluster = nb[static_cast<size_t>(i)];
  }
  r.mean = mean;
  r.metric = metric;
  r.engine = engine;
  r.shards = 1;
  r.cluster_names.reserve(static_cast<size_t>(k));
  for (int32_t c = 0; c < k; ++c) r.cluster_names.push_back(std::to_string(raw[static_cast<size_t>(c)]));
  r.wall_time_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

/// Convenience overload on a per-thread default context for device 0 (fp32 or fp64).
template <typename T>
inline SilhouetteReport compute_silhouette(const std::vector<T>& X, const std::vector<int32_t>& labels,
                                           int32_t d, Metric metric, Engine engine = Engine::Fast,
                                           int shards = 0) {
  if (d <= 0 || X.size() != labels.size() * static_cast<size_t>(d))
    throw ValidationError("feature matrix has " + std::to_string(X.size()) + " values, expected " +
                          std::to_string(labels.size()) + " x " + std::to_string(d));
  thread_local Context ctx(0);
  return compute_silhouette(ctx, X.data(), labels.data(), static_cast<int64_t>(labels.size()), d, metric,
                            engine, shards);
}

}  // namespace fsil
