// oracle/ref_entry.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C entry points over the reference fastsil library compiled UNMODIFIED from
// /root/reference/proj/src (types, dataset, squared_euclidean, cosine, engine,
// report, naive, blobs, csv, report_io .cpp) against oracle/eigen_shim.  Built by
// `make -C oracle ref` into oracle/_ref/libfsil_ref.so, which is git-ignored and
// travels to the GPU box with the snapshot.  Used only by tests/ (to pin the
// restatement in fsil_oracle.cpp bit for bit) and by bench.py's reference arm.
//
// Signatures mirror oracle/fsil_oracle.h (orc_* -> ref_*), so the same ctypes
// binding drives both.  Status codes: 0 ok, 1 IoError, 2 ValidationError,
// 3 std::invalid_argument, 6 anything else.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "fastsil/blobs.hpp"
#include "fastsil/csv.hpp"
#include "fastsil/engine.hpp"
#include "fastsil/report_io.hpp"

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
    return 0;
  } catch (const fastsil::IoError& e) {
    put_err(err, errlen, e.what());
    return 1;
  } catch (const fastsil::ValidationError& e) {
    put_err(err, errlen, e.what());
    return 2;
  } catch (const std::invalid_argument& e) {
    put_err(err, errlen, e.what());
    return 3;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 6;
  }
}

fastsil::Metric to_metric(int m) {
  switch (m) {
    case 0: return fastsil::Metric::SquaredEuclidean;
    case 1: return fastsil::Metric::Cosine;
    case 2: return fastsil::Metric::Euclidean;
  }
  throw std::invalid_argument("unknown metric");
}

void emit(const fastsil::SilhouetteReport& r, double* a, double* b, double* s, int32_t* own,
          int32_t* nb, double* mean, int32_t* k_out, int32_t* dense_to_raw, double* wall_ms) {
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
  if (k_out) *k_out = static_cast<int32_t>(r.cluster_names.size());
  if (dense_to_raw)
    for (size_t k = 0; k < r.cluster_names.size(); ++k) dense_to_raw[k] = std::stoi(r.cluster_names[k]);
  if (wall_ms) *wall_ms = r.wall_time_ms;
}

// N x D row-major == the reference's D x N column-major Matrix, byte for byte.
template <typename T>
fastsil::Matrix to_matrix(const T* X, int64_t n, int64_t d) {
  if (n < 0 || d < 0) throw std::invalid_argument("negative shape");
  fastsil::Matrix m(d, n);
  double* p = m.data();
  for (int64_t j = 0; j < n * d; ++j) p[j] = static_cast<double>(X[j]);
  return m;
}

template <typename T>
int silhouette(int metric, int engine, const T* X, const int32_t* labels, int64_t n, int64_t d,
               int shards, double* a, double* b, double* s, int32_t* own, int32_t* nb, double* mean,
               int32_t* k_out, int32_t* d2r, double* wall_ms, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    std::vector<int> lab(labels, labels + n);
    const fastsil::Dataset ds = fastsil::validate_and_densify(to_matrix(X, n, d), lab);
    const fastsil::SilhouetteReport r = fastsil::compute_silhouette(
        ds, to_metric(metric), engine == 1 ? fastsil::Engine::Naive : fastsil::Engine::Fast, shards);
    emit(r, a, b, s, own, nb, mean, k_out, d2r, wall_ms);
  });
}

}  // namespace

extern "C" {

// compute_silhouette(validate_and_densify(X, labels), metric, engine, shards)
// (engine.cpp:76-92, dataset.cpp:63-68).
int ref_silhouette(int metric, int engine, const double* X, const int32_t* labels, int64_t n,
                   int64_t d, int shards, double* a, double* b, double* s, int32_t* own,
                   int32_t* nb, double* mean, int32_t* k_out, int32_t* d2r, double* wall_ms,
                   char* err, size_t errlen) {
  return silhouette(metric, engine, X, labels, n, d, shards, a, b, s, own, nb, mean, k_out, d2r,
                    wall_ms, err, errlen);
}

int ref_silhouette_f32(int metric, int engine, const float* X, const int32_t* labels, int64_t n,
                       int64_t d, int shards, double* a, double* b, double* s, int32_t* own,
                       int32_t* nb, double* mean, int32_t* k_out, int32_t* d2r, double* wall_ms,
                       char* err, size_t errlen) {
  return silhouette(metric, engine, X, labels, n, d, shards, a, b, s, own, nb, mean, k_out, d2r,
                    wall_ms, err, errlen);
}

// plan_shards (engine.cpp:8-25).
int ref_plan_shards(int64_t n, int requested, int64_t* ranges, int* num_shards, char* err,
                    size_t errlen) {
  return guarded(err, errlen, [&] {
    const fastsil::ShardPlan p = fastsil::plan_shards(n, requested);
    if (num_shards) *num_shards = p.num_shards;
    for (size_t i = 0; i < p.ranges.size(); ++i) {
      ranges[2 * i] = p.ranges[i].first;
      ranges[2 * i + 1] = p.ranges[i].second;
    }
  });
}

// assemble_score (report.cpp:7-14).
int ref_assemble_score(double a, double b, double* s, char* err, size_t errlen) {
  return guarded(err, errlen, [&] { *s = fastsil::assemble_score(a, b); });
}

// generate_blobs (blobs.cpp:25-54): X[n*d] row-major, dense labels[n].
int ref_generate_blobs(int64_t n, int64_t d, int64_t k, double spread, double separation,
                       uint64_t seed, double* X, int32_t* labels, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    fastsil::BlobSpec spec;
    spec.n = n;
    spec.d = d;
    spec.k = k;
    spec.spread = spread;
    spec.separation = separation;
    spec.seed = seed;
    const fastsil::Dataset ds = fastsil::generate_blobs(spec);
    std::memcpy(X, ds.points().data(), sizeof(double) * static_cast<size_t>(n * d));
    for (int64_t i = 0; i < n; ++i) labels[i] = ds.label(i);
  });
}

// read_csv_text (csv.cpp:54-159) -> shape, row-major X, dense labels, and the
// cluster names joined by '\n'.  Call with X == NULL first to get the shape.
int ref_read_csv_text(const char* text, char delimiter, int label_index, const char* label_name,
                      int has_header /* -1 auto, 0, 1 */, int64_t* n_out, int64_t* d_out, double* X,
                      int32_t* labels, char* names, size_t names_len, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    fastsil::CsvSchema schema;
    schema.delimiter = delimiter;
    schema.label_index = label_index;
    schema.label_name = label_name ? label_name : "";
    if (has_header >= 0) schema.has_header = has_header != 0;
    const fastsil::Dataset ds = fastsil::read_csv_text(text, schema);
    *n_out = ds.num_points();
    *d_out = ds.dims();
    if (!X) return;
    std::memcpy(X, ds.points().data(), sizeof(double) * static_cast<size_t>(*n_out * *d_out));
    for (int64_t i = 0; i < *n_out; ++i) labels[i] = ds.label(i);
    std::string joined;
    for (const auto& nm : ds.cluster_names()) joined += nm + "\n";
    put_err(names, names_len, joined.c_str());
  });
}

// compute_silhouette + write_report (report_io.cpp:53-68) into `out` (format 0
// csv, 1 jsonl); *out_len receives the full length.
int ref_score_report(int metric, const double* X, const int32_t* labels, int64_t n, int64_t d,
                     int format, char* out, size_t out_cap, size_t* out_len, char* err,
                     size_t errlen) {
  return guarded(err, errlen, [&] {
    std::vector<int> lab(labels, labels + n);
    const fastsil::Dataset ds = fastsil::validate_and_densify(to_matrix(X, n, d), lab);
    const fastsil::SilhouetteReport r =
        fastsil::compute_silhouette(ds, to_metric(metric), fastsil::Engine::Fast, 1);
    std::ostringstream os;
    fastsil::write_report(r, os, format == 1 ? fastsil::ReportFormat::Jsonl : fastsil::ReportFormat::Csv);
    const std::string str = os.str();
    *out_len = str.size();
    if (out && out_cap) {
      const size_t m = std::min(out_cap - 1, str.size());
      std::memcpy(out, str.data(), m);
      out[m] = '\0';
    }
  });
}

int ref_default_shards(void) { return fastsil::default_shards(); }

}  // extern "C"
