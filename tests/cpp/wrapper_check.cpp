// wrapper_check.cpp -- exercises include/fsil/silhouette.hpp the way a fastsil caller would.
//   wrapper_check no-device   : Context construction must throw CudaError (no CPU fallback)
//   wrapper_check golden      : SPEC known answers (square -> 31/33, orthogonal cosine -> 1),
//                               error mapping, plan_shards / assemble_score
// Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <sstream>

#include "fsil/report_io.hpp"
#include "fsil/silhouette.hpp"

static int failures = 0;
#define CHECK(...)                                                    \
  do {                                                                \
    if (!(__VA_ARGS__)) {                                             \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static bool near(double x, double y, double tol) { return std::fabs(x - y) <= tol; }

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "golden";
  // host-only entries work without a device
  const fsil::ShardPlan plan = fsil::plan_shards(10, 3);
  CHECK(plan.num_shards == 3 && plan.ranges[0] == std::make_pair<int64_t, int64_t>(0, 4) &&
        plan.ranges[2] == std::make_pair<int64_t, int64_t>(7, 10));
  CHECK(fsil::assemble_score(1.0, 16.5) == 1.0 - 1.0 / 16.5);
  CHECK(fsil::assemble_score(0.0, 0.0) == 0.0);
  bool threw = false;
  try {
    fsil::assemble_score(-1.0, 1.0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  CHECK(fsil::parse_metric("sqeuclid") == fsil::Metric::SquaredEuclidean);
  // report emission (report_io.cpp): 17 significant digits, csv + summary, jsonl
  {
    fsil::SilhouetteReport rep;
    rep.scores.push_back({1.0, 16.5, 1.0 - 1.0 / 16.5, 0, 1});
    rep.mean = 0.1;
    std::ostringstream csv, js;
    fsil::write_report(rep, csv, fsil::ReportFormat::Csv);
    fsil::write_report(rep, js, fsil::ReportFormat::Jsonl);
    CHECK(csv.str() == "index,own_cluster,neighbour_cluster,a,b,s\n0,0,1,1,16.5,0.93939393939393945\n"
                       "# summary: mean=0.10000000000000001 metric=squared_euclidean engine=fast shards=1 "
                       "wall_time_ms=0\n");
    CHECK(js.str().rfind("{\"index\":0,\"own\":0,\"neighbour\":1,\"a\":1,\"b\":16.5,\"s\":0.93939393939393945}\n", 0) == 0);
  }
  CHECK(fsil::metric_name(fsil::Metric::Cosine) == "cosine");

  if (mode == "no-device") {
    threw = false;
    try {
      fsil::Context ctx(0);
    } catch (const fsil::CudaError& e) {
      threw = true;
      std::printf("no device: %s\n", e.what());
    }
    CHECK(threw);
  } else {
    fsil::Context ctx(0);
    // SPEC known answer: unit-spaced square pairs 4 apart -> every s_i = 31/33
    const std::vector<float> sq = {0, 0, 0, 1, 4, 0, 4, 1};
    const std::vector<int32_t> lab = {7, 7, 3, 3};
    fsil::SilhouetteReport r = fsil::compute_silhouette(ctx, sq.data(), lab.data(), 4, 2, fsil::Metric::SquaredEuclidean);
    CHECK(near(r.mean, 31.0 / 33.0, 1e-12));
    for (const auto& p : r.scores) {
      CHECK(near(p.a, 1.0, 1e-12) && near(p.b, 16.5, 1e-12) && near(p.s, 31.0 / 33.0, 1e-12));
    }
    CHECK(r.scores[0].own_cluster == 0 && r.scores[0].neighbour_cluster == 1 && r.scores[2].own_cluster == 1);
    CHECK(r.cluster_names.size() == 2 && r.cluster_names[0] == "7" && r.cluster_names[1] == "3");
    // the same known answer through the fp64 front end (the reference's Matrix type)
    const std::vector<double> sq64 = {0, 0, 0, 1, 4, 0, 4, 1};
    r = fsil::compute_silhouette(ctx, sq64.data(), lab.data(), 4, 2, fsil::Metric::SquaredEuclidean);
    CHECK(near(r.mean, 31.0 / 33.0, 1e-12) && near(r.scores[3].b, 16.5, 1e-12));
    // orthogonal cosine clusters -> mean 1
    const std::vector<float> co = {1, 0, 2, 0, 0, 1, 0, 3};
    r = fsil::compute_silhouette(ctx, co.data(), lab.data(), 4, 2, fsil::Metric::Cosine);
    CHECK(near(r.mean, 1.0, 1e-12));
    // error mapping: one cluster -> ValidationError; plain euclidean on the fast engine too
    const std::vector<int32_t> one = {5, 5, 5, 5};
    threw = false;
    try {
      fsil::compute_silhouette(ctx, sq.data(), one.data(), 4, 2, fsil::Metric::SquaredEuclidean);
    } catch (const fsil::ValidationError& e) {
      threw = std::strstr(e.what(), "single cluster") != nullptr;
    }
    CHECK(threw);
    threw = false;
    try {
      fsil::compute_silhouette(ctx, sq.data(), lab.data(), 4, 2, fsil::Metric::Euclidean);
    } catch (const fsil::ValidationError&) {
      threw = true;
    }
    CHECK(threw);
    // the naive engine: the same known answer, and plain Euclidean (naive only):
    // a = 1, b = (4 + sqrt(17)) / 2 for every point of the square
    r = fsil::compute_silhouette(ctx, sq.data(), lab.data(), 4, 2, fsil::Metric::SquaredEuclidean, fsil::Engine::Naive);
    CHECK(near(r.mean, 31.0 / 33.0, 1e-12) && r.engine == fsil::Engine::Naive);
    r = fsil::compute_silhouette(ctx, sq.data(), lab.data(), 4, 2, fsil::Metric::Euclidean, fsil::Engine::Naive);
    const double be = (4.0 + std::sqrt(17.0)) / 2.0;
    CHECK(near(r.scores[0].a, 1.0, 1e-12) && near(r.scores[0].b, be, 1e-12) && near(r.mean, 1.0 - 1.0 / be, 1e-12));
    std::printf("golden: mean %.17g, K %zu, path %d\n", 31.0 / 33.0, r.cluster_names.size(), ctx.stats().path);
  }
  if (failures) std::fprintf(stderr, "%d check(s) failed\n", failures);
  return failures ? 1 : 0;
}
