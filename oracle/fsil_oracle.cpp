// fsil_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see fsil_oracle.h).
//
// Faithful CPU restatement of the reference fastsil fast path and its naive
// oracle, written without Eigen.  Every function names the reference
// file:line it restates (paths under /root/reference/proj).  Build flags
// follow the reference (proj/CMakeLists.txt:8-10,20): -O3 -DNDEBUG -std=c++20,
// no -march, no OpenMP; threads are std::thread as in engine.cpp:34-55.

#include "fsil_oracle.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

namespace orc {

using Index = int64_t;

// ---- types.hpp:20-50 ------------------------------------------------------
enum class Metric { SquaredEuclidean, Cosine, Euclidean };
enum class Engine { Fast, Naive };

struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- dataset.hpp:14-40 -----------------------------------------------------
// D x N column-major fp64 == N x D row-major: point i is the contiguous run
// pts[i*D .. i*D+D).
struct Dataset {
  std::vector<double> pts;
  Index n = 0, d = 0;
  std::vector<int> labels;          // dense
  std::vector<Index> sizes;         // cluster_sizes
  std::vector<std::string> names;   // cluster_names, dense order
  Index num_points() const { return n; }
  Index dims() const { return d; }
  Index num_clusters() const { return static_cast<Index>(sizes.size()); }
  const double* point(Index i) const { return pts.data() + i * d; }
  int label(Index i) const { return labels[static_cast<size_t>(i)]; }
};

// squaredNorm / dot / norm as the reference's Eigen computes them (types.hpp:3;
// Eigen 3.4.0, restated -- Eigen is not installed here).  The reference is built
// without -march (proj/CMakeLists.txt:20), so Eigen reduces with SSE2 Packet2d in
// redux_impl<LinearVectorizedTraversal, NoUnrolling> (Eigen/src/Core/Redux.h):
// four interleaved partial sums over 4*floor(n/4) terms -- lane j sums terms
// j, j+4, j+8, ... -- folded as (s0+s2, s1+s3), plus one more pair when n mod 4 >= 2,
// then lane 0 + lane 1, then the odd tail term.  sum() of nothing is 0.  Pinned
// bit for bit against the reference sources compiled by oracle/Makefile `ref`.
template <typename Term>
static double eigen_redux_sum(Index n, Term term) {
  if (n == 0) return 0.0;
  const Index pairs_end = (n / 2) * 2, quads_end = (n / 4) * 4;
  if (pairs_end == 0) return term(0);
  double s0 = term(0), s1 = term(1);
  if (pairs_end > 2) {
    double s2 = term(2), s3 = term(3);
    for (Index i = 4; i < quads_end; i += 4) {
      s0 += term(i);
      s1 += term(i + 1);
      s2 += term(i + 2);
      s3 += term(i + 3);
    }
    s0 += s2;
    s1 += s3;
    if (pairs_end > quads_end) {
      s0 += term(quads_end);
      s1 += term(quads_end + 1);
    }
  }
  double res = s0 + s1;
  for (Index i = pairs_end; i < n; ++i) res += term(i);
  return res;
}
static double sq_norm(const double* x, Index d) {  // cwiseAbs2().sum()
  return eigen_redux_sum(d, [x](Index l) { return x[l] * x[l]; });
}
static double dot(const double* x, const double* y, Index d) {  // binaryExpr(conj_prod).sum()
  return eigen_redux_sum(d, [x, y](Index l) { return x[l] * y[l]; });
}
static double sq_dist(const double* p, const double* q, Index d) {  // (p - q).squaredNorm()
  return eigen_redux_sum(d, [p, q](Index l) {
    const double t = p[l] - q[l];
    return t * t;
  });
}
static double norm(const double* x, Index d) { return std::sqrt(sq_norm(x, d)); }

// locate_non_finite: dataset.cpp:13-22 (column-by-column = row-major scan).
static std::string locate_non_finite(const std::vector<double>& pts, Index n, Index d) {
  for (Index i = 0; i < n; ++i)
    for (Index l = 0; l < d; ++l)
      if (!std::isfinite(pts[static_cast<size_t>(i * d + l)]))
        return "point " + std::to_string(i) + ", dimension " + std::to_string(l);
  return "unknown position";
}

// validate_and_densify(Matrix, vector<string>): dataset.cpp:26-61.
static Dataset validate_and_densify(std::vector<double> pts, Index n, Index d,
                                    const std::vector<std::string>& labels) {
  if (static_cast<size_t>(n) != labels.size())
    throw ValidationError("label count (" + std::to_string(labels.size()) +
                          ") does not match point count (" + std::to_string(n) + ")");
  if (n < 2) throw ValidationError("dataset needs at least 2 points, got " + std::to_string(n));
  if (d < 1) throw ValidationError("dataset needs at least 1 feature dimension");
  bool finite = true;
  for (double v : pts) finite = finite && std::isfinite(v);
  if (!finite) throw ValidationError("non-finite feature value at " + locate_non_finite(pts, n, d));

  Dataset ds;
  ds.n = n;
  ds.d = d;
  ds.labels.resize(labels.size());
  std::unordered_map<std::string, int> dense;  // first appearance -> dense id (:41-51)
  dense.reserve(labels.size());
  for (size_t i = 0; i < labels.size(); ++i) {
    auto [it, inserted] = dense.try_emplace(labels[i], static_cast<int>(ds.names.size()));
    if (inserted) {
      ds.names.push_back(labels[i]);
      ds.sizes.push_back(0);
    }
    ds.labels[i] = it->second;
    ++ds.sizes[static_cast<size_t>(it->second)];
  }
  if (ds.names.size() < 2)
    throw ValidationError("silhouette undefined for a single cluster: need K >= 2, got K = " +
                          std::to_string(ds.names.size()));
  ds.pts = std::move(pts);
  return ds;
}

// int overload: dataset.cpp:63-68 (labels stringified, then densified).
static Dataset validate_and_densify(std::vector<double> pts, Index n, Index d,
                                    const int32_t* labels) {
  std::vector<std::string> names;
  names.reserve(static_cast<size_t>(n));
  for (Index i = 0; i < n; ++i) names.push_back(std::to_string(labels[i]));
  return validate_and_densify(std::move(pts), n, d, names);
}

// ---- report.hpp:10-26, report.cpp:7-47 ------------------------------------
struct PointScore {
  double a = 0.0, b = 0.0, s = 0.0;
  int own_cluster = -1, neighbour_cluster = -1;
};

struct Report {
  std::vector<PointScore> scores;
  double mean = 0.0;
  double wall_time_ms = 0.0;
  std::vector<std::string> names;
};

static double assemble_score(double a, double b) {  // report.cpp:7-14
  if (a < 0.0 || b < 0.0)
    throw std::invalid_argument("assemble_score: negative mean distance (a=" + std::to_string(a) +
                                ", b=" + std::to_string(b) + ")");
  if (a == 0.0 && b == 0.0) return 0.0;
  return a <= b ? 1.0 - a / b : b / a - 1.0;
}

static PointScore make_point_score(double own_mean, double min_foreign, int own, int nb,
                                   bool singleton) {  // report.cpp:16-30
  PointScore p;
  p.own_cluster = own;
  p.neighbour_cluster = nb;
  p.b = min_foreign;
  if (singleton) {
    p.a = 0.0;
    p.s = 0.0;
  } else {
    p.a = own_mean;
    p.s = assemble_score(own_mean, min_foreign);
  }
  return p;
}

static Report finalize_report(std::vector<PointScore> scores,
                              std::vector<std::string> names) {  // report.cpp:32-47
  if (scores.empty()) throw ValidationError("cannot finalize an empty report (N >= 2 required)");
  double sum = 0.0;  // left-to-right, dataset order
  for (const PointScore& p : scores) sum += p.s;
  Report r;
  r.mean = sum / static_cast<double>(scores.size());
  r.scores = std::move(scores);
  r.names = std::move(names);
  return r;
}

// ---- squared_euclidean.hpp:20-65, squared_euclidean.cpp:9-108 ---------------
static void check_range(Index begin, Index end, Index n) {  // sqE.cpp:11-17
  if (begin < 0 || end > n || begin > end)
    throw std::invalid_argument("point range [" + std::to_string(begin) + ", " +
                                std::to_string(end) + ") outside dataset of size " +
                                std::to_string(n));
}

static void check_label(int label, Index k, Index point) {  // sqE.cpp:19-25
  if (label < 0 || label >= k)
    throw ValidationError("cluster label " + std::to_string(label) + " of point " +
                          std::to_string(point) + " outside [0, " + std::to_string(k) + ")");
}

struct SqStats {  // SqEuclidClusterStats
  Index k = 0, d = 0;
  std::vector<int64_t> counts;   // K  (IntVector in the reference)
  std::vector<double> psi;       // K  sq_norm_sums
  std::vector<double> y;         // K x D point_sums, cluster-major (col k of D x K)
  static SqStats zero(Index k, Index d) {
    SqStats s;
    s.k = k;
    s.d = d;
    s.counts.assign(static_cast<size_t>(k), 0);
    s.psi.assign(static_cast<size_t>(k), 0.0);
    s.y.assign(static_cast<size_t>(k * d), 0.0);
    return s;
  }
};

struct SqPolicy {
  using Stats = SqStats;
  static constexpr Metric metric = Metric::SquaredEuclidean;
  static void precheck(const Dataset&) {}
  // partial_cluster_stats: sqE.cpp:37-54
  static Stats partial(const Dataset& ds, Index begin, Index end) {
    check_range(begin, end, ds.n);
    Stats st = Stats::zero(ds.num_clusters(), ds.d);
    for (Index i = begin; i < end; ++i) {
      const int k = ds.label(i);
      check_label(k, st.k, i);
      const double* x = ds.point(i);
      st.counts[k] += 1;
      st.psi[k] += sq_norm(x, ds.d);
      double* yk = st.y.data() + k * ds.d;
      for (Index l = 0; l < ds.d; ++l) yk[l] += x[l];
    }
    return st;
  }
  // merge_stats: sqE.cpp:56-63
  static void merge(Stats& into, const Stats& from) {
    if (into.k != from.k || into.d != from.d)
      throw ValidationError("cannot merge cluster stats of mismatched shape");
    for (Index k = 0; k < into.k; ++k) {
      into.counts[k] += from.counts[k];
      into.psi[k] += from.psi[k];
    }
    for (size_t j = 0; j < into.y.size(); ++j) into.y[j] += from.y[j];
  }
  // mean_dist_to_cluster: sqE.cpp:65-82
  static double mean_dist(double xi, const double* x, const Stats& st, Index k, bool exclude_self) {
    const int64_t count = st.counts[k];
    if (count < 1) throw std::invalid_argument("mean distance to an empty cluster");
    const double n = static_cast<double>(count);
    const double cross = dot(st.y.data() + k * st.d, x, st.d);
    double mean;
    if (exclude_self) {
      if (count < 2)
        throw std::invalid_argument(
            "exclude_self needs a cluster of >= 2 members; apply the singleton convention instead");
      mean = (n * xi + st.psi[k] - 2.0 * cross) / (n - 1.0);
    } else {
      mean = xi + st.psi[k] / n - 2.0 * cross / n;
    }
    return std::max(0.0, mean);
  }
  // score_range: sqE.cpp:84-108
  static void score(const Dataset& ds, const Stats& st, Index begin, Index end,
                    std::span<PointScore> out) {
    check_range(begin, end, ds.n);
    for (Index i = begin; i < end; ++i) {
      const double* x = ds.point(i);
      const double xi = sq_norm(x, ds.d);
      const int own = ds.label(i);
      const bool singleton = st.counts[own] == 1;
      double best = std::numeric_limits<double>::infinity();
      Index nb = -1;
      for (Index k = 0; k < st.k; ++k) {
        if (k == own) continue;
        const double m = mean_dist(xi, x, st, k, false);
        if (m < best) {  // strict: ties keep the lowest dense index
          best = m;
          nb = k;
        }
      }
      const double a = singleton ? 0.0 : mean_dist(xi, x, st, own, true);
      out[static_cast<size_t>(i)] = make_point_score(a, best, own, static_cast<int>(nb), singleton);
    }
  }
};

// ---- cosine.hpp:16-59, cosine.cpp:9-123 ------------------------------------
[[noreturn]] static void throw_zero_norm(Index point) {  // cosine.cpp:19-22
  throw ValidationError("cosine distance undefined for zero vector (point " +
                        std::to_string(point) + ")");
}

struct CosStats {  // CosineClusterStats
  Index k = 0, d = 0;
  std::vector<int64_t> counts;
  std::vector<double> omega;  // K x D unit_sums, cluster-major
  static CosStats zero(Index k, Index d) {
    CosStats s;
    s.k = k;
    s.d = d;
    s.counts.assign(static_cast<size_t>(k), 0);
    s.omega.assign(static_cast<size_t>(k * d), 0.0);
    return s;
  }
};

struct CosPolicy {
  using Stats = CosStats;
  static constexpr Metric metric = Metric::Cosine;
  // require_nonzero_norms: cosine.cpp:119-123
  static void precheck(const Dataset& ds) {
    for (Index i = 0; i < ds.n; ++i)
      if (norm(ds.point(i), ds.d) == 0.0) throw_zero_norm(i);
  }
  // partial_unit_sums: cosine.cpp:39-61
  static Stats partial(const Dataset& ds, Index begin, Index end) {
    check_range(begin, end, ds.n);
    Stats st = Stats::zero(ds.num_clusters(), ds.d);
    for (Index i = begin; i < end; ++i) {
      const int k = ds.label(i);
      if (k < 0 || k >= st.k)
        throw ValidationError("cluster label " + std::to_string(k) + " of point " +
                              std::to_string(i) + " outside [0, " + std::to_string(st.k) + ")");
      const double* x = ds.point(i);
      const double nrm = norm(x, ds.d);
      if (nrm == 0.0) throw_zero_norm(i);
      st.counts[k] += 1;
      double* ok = st.omega.data() + k * ds.d;
      for (Index l = 0; l < ds.d; ++l) ok[l] += x[l] / nrm;
    }
    return st;
  }
  // merge_stats: cosine.cpp:63-69
  static void merge(Stats& into, const Stats& from) {
    if (into.k != from.k || into.d != from.d)
      throw ValidationError("cannot merge cluster stats of mismatched shape");
    for (Index k = 0; k < into.k; ++k) into.counts[k] += from.counts[k];
    for (size_t j = 0; j < into.omega.size(); ++j) into.omega[j] += from.omega[j];
  }
  // mean_dist_to_cluster: cosine.cpp:71-88
  static double mean_dist(const double* unit, const Stats& st, Index k, bool exclude_self) {
    const int64_t count = st.counts[k];
    if (count < 1) throw std::invalid_argument("mean distance to an empty cluster");
    const double n = static_cast<double>(count);
    const double cross = dot(st.omega.data() + k * st.d, unit, st.d);
    double mean;
    if (exclude_self) {
      if (count < 2)
        throw std::invalid_argument(
            "exclude_self needs a cluster of >= 2 members; apply the singleton convention instead");
      mean = (n - cross) / (n - 1.0);
    } else {
      mean = 1.0 - cross / n;
    }
    return std::clamp(mean, 0.0, 2.0);
  }
  // score_range: cosine.cpp:90-117
  static void score(const Dataset& ds, const Stats& st, Index begin, Index end,
                    std::span<PointScore> out) {
    check_range(begin, end, ds.n);
    std::vector<double> unit(static_cast<size_t>(ds.d));
    for (Index i = begin; i < end; ++i) {
      const double* x = ds.point(i);
      const double nrm = norm(x, ds.d);
      if (nrm == 0.0) throw_zero_norm(i);
      for (Index l = 0; l < ds.d; ++l) unit[l] = x[l] / nrm;
      const int own = ds.label(i);
      const bool singleton = st.counts[own] == 1;
      double best = std::numeric_limits<double>::infinity();
      Index nb = -1;
      for (Index k = 0; k < st.k; ++k) {
        if (k == own) continue;
        const double m = mean_dist(unit.data(), st, k, false);
        if (m < best) {
          best = m;
          nb = k;
        }
      }
      const double a = singleton ? 0.0 : mean_dist(unit.data(), st, own, true);
      out[static_cast<size_t>(i)] = make_point_score(a, best, own, static_cast<int>(nb), singleton);
    }
  }
};

// ---- engine.hpp:18-115, engine.cpp:8-92 ------------------------------------
struct ShardPlan {
  int num_shards = 1;
  std::vector<std::pair<Index, Index>> ranges;
};

static ShardPlan plan_shards(Index n, int requested) {  // engine.cpp:8-25
  if (n < 1) throw std::invalid_argument("plan_shards: need at least one point");
  if (requested < 1) throw std::invalid_argument("plan_shards: need at least one worker");
  const Index w = std::min<Index>(requested, n);
  ShardPlan plan;
  plan.num_shards = static_cast<int>(w);
  const Index base = n / w, extra = n % w;
  Index begin = 0;
  for (Index s = 0; s < w; ++s) {
    const Index size = base + (s < extra ? 1 : 0);
    plan.ranges.emplace_back(begin, begin + size);
    begin += size;
  }
  return plan;
}

static int default_shards() {  // engine.cpp:27-30
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : static_cast<int>(hw);
}

constexpr Index kMaxAggregationBlocks = 256;    // engine.hpp:34
constexpr Index kMinAggregationBlockSize = 512; // engine.hpp:35
static Index aggregation_block_size(Index n) {  // engine.hpp:37-40
  const Index even = (n + kMaxAggregationBlocks - 1) / kMaxAggregationBlocks;
  return std::max(kMinAggregationBlockSize, even);
}

// run_workers: engine.cpp:34-55 (lowest-index exception rethrown).
static void run_workers(int count, const std::function<void(int)>& body) {
  if (count <= 1) {
    body(0);
    return;
  }
  std::vector<std::exception_ptr> errors(static_cast<size_t>(count));
  std::vector<std::thread> workers;
  workers.reserve(static_cast<size_t>(count));
  for (int w = 0; w < count; ++w)
    workers.emplace_back([&, w] {
      try {
        body(w);
      } catch (...) {
        errors[static_cast<size_t>(w)] = std::current_exception();
      }
    });
  for (auto& t : workers) t.join();
  for (const auto& e : errors)
    if (e) std::rethrow_exception(e);
}

// aggregate_cluster_stats: engine.hpp:50-80 (N-only blocks, ascending fold).
template <typename Policy>
static typename Policy::Stats aggregate(const Dataset& ds, int workers) {
  const Index n = ds.n;
  const Index block = aggregation_block_size(n);
  const Index nblocks = (n + block - 1) / block;
  std::vector<typename Policy::Stats> partials(static_cast<size_t>(nblocks));
  auto run_block = [&](Index b) {
    const Index begin = b * block;
    const Index end = std::min(n, begin + block);
    partials[static_cast<size_t>(b)] = Policy::partial(ds, begin, end);
  };
  const int pool = static_cast<int>(std::min<Index>(workers, nblocks));
  if (pool <= 1) {
    for (Index b = 0; b < nblocks; ++b) run_block(b);
  } else {
    std::atomic<Index> next{0};
    run_workers(pool, [&](int) {
      for (Index b; (b = next.fetch_add(1, std::memory_order_relaxed)) < nblocks;) run_block(b);
    });
  }
  typename Policy::Stats merged = std::move(partials.front());
  for (Index b = 1; b < nblocks; ++b) Policy::merge(merged, partials[static_cast<size_t>(b)]);
  return merged;
}

// score_into: engine.hpp:86-103
template <typename Policy>
static void score_into(const Dataset& ds, const ShardPlan& plan, std::span<PointScore> out) {
  if (static_cast<Index>(out.size()) != ds.n)
    throw std::invalid_argument("score_into: output size must equal the point count");
  Policy::precheck(ds);
  const typename Policy::Stats merged = aggregate<Policy>(ds, plan.num_shards);
  if (plan.num_shards <= 1) {
    Policy::score(ds, merged, 0, ds.n, out);
  } else {
    run_workers(static_cast<int>(plan.ranges.size()), [&](int s) {
      const auto [begin, end] = plan.ranges[static_cast<size_t>(s)];
      Policy::score(ds, merged, begin, end, out);
    });
  }
}

// run_two_phase: engine.hpp:105-115 (the reference's timed window).
template <typename Policy>
static Report run_two_phase(const Dataset& ds, const ShardPlan& plan) {
  const auto start = std::chrono::steady_clock::now();
  std::vector<PointScore> scores(static_cast<size_t>(ds.n));
  score_into<Policy>(ds, plan, scores);
  Report r = finalize_report(std::move(scores), ds.names);
  r.wall_time_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
  return r;
}

// ---- naive.cpp:12-71 --------------------------------------------------------
static double pairwise_distance(const double* p, const double* q, Index d, Metric metric) {
  switch (metric) {
    case Metric::SquaredEuclidean:
      return sq_dist(p, q, d);
    case Metric::Euclidean:
      return std::sqrt(sq_dist(p, q, d));
    case Metric::Cosine: {
      const double np = norm(p, d), nq = norm(q, d);
      if (np == 0.0 || nq == 0.0) throw ValidationError("cosine distance undefined for zero vector");
      return 1.0 - dot(p, q, d) / (np * nq);
    }
  }
  throw std::invalid_argument("unknown metric");
}

static Report naive_silhouette(const Dataset& ds, Metric metric) {
  if (metric == Metric::Cosine) CosPolicy::precheck(ds);
  const auto start = std::chrono::steady_clock::now();
  const Index n = ds.n, k = ds.num_clusters();
  std::vector<PointScore> scores(static_cast<size_t>(n));
  std::vector<double> sums(static_cast<size_t>(k));
  for (Index i = 0; i < n; ++i) {
    std::fill(sums.begin(), sums.end(), 0.0);
    const double* p = ds.point(i);
    for (Index j = 0; j < n; ++j) {
      if (j == i) continue;
      sums[ds.label(j)] += pairwise_distance(p, ds.point(j), ds.d, metric);
    }
    const int own = ds.label(i);
    const Index own_size = ds.sizes[own];
    const bool singleton = own_size == 1;
    const double a = singleton ? 0.0 : sums[own] / static_cast<double>(own_size - 1);
    double best = std::numeric_limits<double>::infinity();
    Index nb = -1;
    for (Index c = 0; c < k; ++c) {
      if (c == own) continue;
      const double m = sums[c] / static_cast<double>(ds.sizes[c]);
      if (m < best) {
        best = m;
        nb = c;
      }
    }
    scores[static_cast<size_t>(i)] = make_point_score(a, best, own, static_cast<int>(nb), singleton);
  }
  Report r = finalize_report(std::move(scores), ds.names);
  r.wall_time_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
  return r;
}

// compute_silhouette: engine.cpp:76-92
static Report compute_silhouette(const Dataset& ds, Metric metric, Engine engine, int shards) {
  if (engine == Engine::Naive) return naive_silhouette(ds, metric);
  const int requested = shards > 0 ? shards : default_shards();
  const ShardPlan plan = plan_shards(ds.n, requested);
  switch (metric) {
    case Metric::SquaredEuclidean:
      return run_two_phase<SqPolicy>(ds, plan);
    case Metric::Cosine:
      return run_two_phase<CosPolicy>(ds, plan);
    case Metric::Euclidean:
      break;
  }
  throw ValidationError(
      "no fast engine for plain euclidean distance (no aggregable decomposition); "
      "use the naive engine");
}

}  // namespace orc

// ---- C ABI -------------------------------------------------------------------
namespace {

void put_err(char* err, size_t errlen, const char* msg) {
  if (err && errlen) {
    std::strncpy(err, msg, errlen - 1);
    err[errlen - 1] = '\0';
  }
}

template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
  try {
    f();
    put_err(err, errlen, "");
    return ORC_OK;
  } catch (const orc::ValidationError& e) {
    put_err(err, errlen, e.what());
    return ORC_ERR_VALIDATION;
  } catch (const std::invalid_argument& e) {
    put_err(err, errlen, e.what());
    return ORC_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return ORC_ERR_INTERNAL;
  }
}

orc::Metric to_metric(int m) {
  switch (m) {
    case ORC_SQEUCLID:
      return orc::Metric::SquaredEuclidean;
    case ORC_COSINE:
      return orc::Metric::Cosine;
    case ORC_EUCLID:
      return orc::Metric::Euclidean;
  }
  throw std::invalid_argument("unknown metric");
}

void emit(const orc::Report& r, double* a, double* b, double* s, int32_t* own, int32_t* nb,
          double* mean, int32_t* k_out, int32_t* dense_to_raw, double* wall_ms) {
  const size_t n = r.scores.size();
  for (size_t i = 0; i < n; ++i) {
    const auto& p = r.scores[i];
    if (a) a[i] = p.a;
    if (b) b[i] = p.b;
    if (s) s[i] = p.s;
    if (own) own[i] = p.own_cluster;
    if (nb) nb[i] = p.neighbour_cluster;
  }
  if (mean) *mean = r.mean;
  if (k_out) *k_out = static_cast<int32_t>(r.names.size());
  if (dense_to_raw)
    for (size_t k = 0; k < r.names.size(); ++k) dense_to_raw[k] = std::stoi(r.names[k]);
  if (wall_ms) *wall_ms = r.wall_time_ms;
}

orc::Dataset densify_f32(const float* X, const int32_t* labels, int64_t n, int64_t d) {
  if (n < 0 || d < 0) throw std::invalid_argument("negative shape");
  std::vector<double> pts(static_cast<size_t>(n * d));
  for (size_t j = 0; j < pts.size(); ++j) pts[j] = static_cast<double>(X[j]);
  return orc::validate_and_densify(std::move(pts), n, d, labels);
}

}  // namespace

extern "C" {

int orc_silhouette(int metric, int engine, const double* X, const int32_t* labels, int64_t n,
                   int64_t d, int shards, double* a, double* b, double* s, int32_t* own,
                   int32_t* neighbour, double* mean, int32_t* k_out, int32_t* dense_to_raw,
                   double* wall_ms, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    if (n < 0 || d < 0) throw std::invalid_argument("negative shape");
    std::vector<double> pts(X, X + n * d);
    const orc::Dataset ds = orc::validate_and_densify(std::move(pts), n, d, labels);
    const orc::Report r = orc::compute_silhouette(
        ds, to_metric(metric), engine == ORC_NAIVE ? orc::Engine::Naive : orc::Engine::Fast, shards);
    emit(r, a, b, s, own, neighbour, mean, k_out, dense_to_raw, wall_ms);
  });
}

int orc_silhouette_f32(int metric, int engine, const float* X, const int32_t* labels, int64_t n,
                       int64_t d, int shards, double* a, double* b, double* s, int32_t* own,
                       int32_t* neighbour, double* mean, int32_t* k_out, int32_t* dense_to_raw,
                       double* wall_ms, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const orc::Dataset ds = densify_f32(X, labels, n, d);
    const orc::Report r = orc::compute_silhouette(
        ds, to_metric(metric), engine == ORC_NAIVE ? orc::Engine::Naive : orc::Engine::Fast, shards);
    emit(r, a, b, s, own, neighbour, mean, k_out, dense_to_raw, wall_ms);
  });
}

int orc_aggregate_f32(int metric, const float* X, const int32_t* labels, int64_t n, int64_t d,
                      int shards, int64_t* counts, double* sums, double* psi, int32_t* k_out,
                      char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const orc::Dataset ds = densify_f32(X, labels, n, d);
    const int w = shards > 0 ? shards : orc::default_shards();
    const int64_t k = ds.num_clusters();
    if (k_out) *k_out = static_cast<int32_t>(k);
    if (to_metric(metric) == orc::Metric::SquaredEuclidean) {
      const auto st = orc::aggregate<orc::SqPolicy>(ds, w);
      for (int64_t c = 0; c < k; ++c) {
        if (counts) counts[c] = st.counts[c];
        if (psi) psi[c] = st.psi[c];
      }
      if (sums) std::copy(st.y.begin(), st.y.end(), sums);
    } else if (to_metric(metric) == orc::Metric::Cosine) {
      orc::CosPolicy::precheck(ds);
      const auto st = orc::aggregate<orc::CosPolicy>(ds, w);
      for (int64_t c = 0; c < k; ++c)
        if (counts) counts[c] = st.counts[c];
      if (sums) std::copy(st.omega.begin(), st.omega.end(), sums);
    } else {
      throw orc::ValidationError("no aggregable decomposition for plain euclidean distance");
    }
  });
}

int orc_aggregate_dense_f32(int metric, const float* X, const int32_t* dense, int64_t n, int64_t d,
                            int32_t k, int shards, int64_t* counts, double* sums, double* psi,
                            char* err, size_t errlen) {
  // Same per-row arithmetic as partial_cluster_stats / partial_unit_sums
  // (sqE.cpp:37-50, cos.cpp:39-57) read straight from fp32 storage (each value
  // widened exactly), same N-only block plan and ascending fold
  // (engine.hpp:37-40,75-78); no fp64 copy of X, so 123 GB inputs fit.
  return guarded(err, errlen, [&] {
    const bool cos = to_metric(metric) == orc::Metric::Cosine;
    const int64_t block = orc::aggregation_block_size(n);
    const int64_t nblocks = (n + block - 1) / block;
    const int64_t S = k * (d + 2);
    std::vector<std::vector<double>> part(static_cast<size_t>(nblocks));
    std::vector<double> xd(static_cast<size_t>(d));
    auto run_block = [&](int64_t b) {
      std::vector<double> st(static_cast<size_t>(S), 0.0);  // [count K][psi K][sums K*D]
      std::vector<double> row(static_cast<size_t>(d));
      const int64_t e = std::min(n, (b + 1) * block);
      for (int64_t i = b * block; i < e; ++i) {
        const int c = dense[i];
        if (c < 0 || c >= k) throw orc::ValidationError("cluster label out of range");
        for (int64_t l = 0; l < d; ++l) row[l] = static_cast<double>(X[i * d + l]);
        const double ss = orc::sq_norm(row.data(), d);
        st[c] += 1.0;
        double* y = st.data() + 2 * k + static_cast<int64_t>(c) * d;
        if (cos) {
          const double nrm = std::sqrt(ss);
          if (nrm == 0.0) orc::throw_zero_norm(i);
          for (int64_t l = 0; l < d; ++l) y[l] += row[l] / nrm;
        } else {
          st[k + c] += ss;
          for (int64_t l = 0; l < d; ++l) y[l] += row[l];
        }
      }
      part[static_cast<size_t>(b)] = std::move(st);
    };
    const int w = shards > 0 ? shards : orc::default_shards();
    std::atomic<int64_t> next{0};
    orc::run_workers(static_cast<int>(std::min<int64_t>(w, nblocks)), [&](int) {
      for (int64_t b; (b = next.fetch_add(1)) < nblocks;) run_block(b);
    });
    std::vector<double> merged = std::move(part[0]);
    for (int64_t b = 1; b < nblocks; ++b)
      for (int64_t j = 0; j < S; ++j) merged[j] += part[b][j];
    for (int32_t c = 0; c < k; ++c) {
      counts[c] = static_cast<int64_t>(merged[c]);
      if (!cos && psi) psi[c] = merged[k + c];
    }
    std::copy(merged.begin() + 2 * k, merged.end(), sums);
  });
}

int orc_score_rows_f32(int metric, const float* X, const int32_t* dense, int64_t n, int64_t d,
                       int32_t k, const int64_t* counts, const double* sums, const double* psi,
                       const int64_t* rows, int64_t m, double* a, double* b, double* s,
                       int32_t* neighbour, char* err, size_t errlen) {
  return orc_score_rows_mt_f32(metric, X, dense, n, d, k, counts, sums, psi, rows, m, 1, a, b, s,
                               neighbour, err, errlen);
}

int orc_score_rows_mt_f32(int metric, const float* X, const int32_t* dense, int64_t n, int64_t d,
                          int32_t k, const int64_t* counts, const double* sums, const double* psi,
                          const int64_t* rows, int64_t m, int threads, double* a, double* b,
                          double* s, int32_t* neighbour, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const bool sq = to_metric(metric) == orc::Metric::SquaredEuclidean;
    orc::SqStats sst;
    orc::CosStats cst;
    if (sq) {
      sst = orc::SqStats::zero(k, d);
      std::copy(counts, counts + k, sst.counts.begin());
      std::copy(psi, psi + k, sst.psi.begin());
      std::copy(sums, sums + k * d, sst.y.begin());
    } else {
      cst = orc::CosStats::zero(k, d);
      std::copy(counts, counts + k, cst.counts.begin());
      std::copy(sums, sums + k * d, cst.omega.begin());
    }
    // Chunks of rows, each a compact dataset of those rows (fp32 widened exactly)
    // against the global stats, scored by the policy's score_range.
    constexpr int64_t kChunk = 4096;
    const int64_t nchunks = (m + kChunk - 1) / kChunk;
    std::atomic<int64_t> next{0};
    auto body = [&](int) {
      orc::Dataset ds;
      ds.d = d;
      ds.sizes.assign(static_cast<size_t>(k), 0);
      std::vector<orc::PointScore> out;
      for (int64_t c; (c = next.fetch_add(1)) < nchunks;) {
        const int64_t j0 = c * kChunk, cm = std::min(m, j0 + kChunk) - j0;
        ds.n = cm;
        ds.pts.resize(static_cast<size_t>(cm * d));
        ds.labels.resize(static_cast<size_t>(cm));
        for (int64_t j = 0; j < cm; ++j) {
          const int64_t r = rows ? rows[j0 + j] : j0 + j;
          if (r < 0 || r >= n) throw std::invalid_argument("row index out of range");
          for (int64_t l = 0; l < d; ++l) ds.pts[j * d + l] = static_cast<double>(X[r * d + l]);
          ds.labels[j] = dense[r];
        }
        out.assign(static_cast<size_t>(cm), orc::PointScore{});
        if (sq) orc::SqPolicy::score(ds, sst, 0, cm, out);
        else orc::CosPolicy::score(ds, cst, 0, cm, out);
        for (int64_t j = 0; j < cm; ++j) {
          if (a) a[j0 + j] = out[j].a;
          if (b) b[j0 + j] = out[j].b;
          if (s) s[j0 + j] = out[j].s;
          if (neighbour) neighbour[j0 + j] = out[j].neighbour_cluster;
        }
      }
    };
    const int w = threads > 0 ? threads : orc::default_shards();
    orc::run_workers(static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(w, nchunks))), body);
  });
}

int orc_plan_shards(int64_t n, int requested, int64_t* ranges, int* num_shards, char* err,
                    size_t errlen) {
  return guarded(err, errlen, [&] {
    const orc::ShardPlan p = orc::plan_shards(n, requested);
    if (num_shards) *num_shards = p.num_shards;
    for (size_t s = 0; s < p.ranges.size(); ++s) {
      ranges[2 * s] = p.ranges[s].first;
      ranges[2 * s + 1] = p.ranges[s].second;
    }
  });
}

int orc_assemble_score(double a, double b, double* s, char* err, size_t errlen) {
  return guarded(err, errlen, [&] { *s = orc::assemble_score(a, b); });
}

int orc_default_shards(void) { return orc::default_shards(); }

}  // extern "C"
