// adagio_b200.hpp -- header-only C++17 facade with the reference's API.
//
// Reproduces the names, structs, defaults and exception types of the
// reference headers proj/include/adagio/{point_cloud,errors,rng,jl,spectral,
// embed,distortion}.hpp on top of the C ABI in adg.h, so a caller such as
// proj/tools/adagio_main.cpp (run_fit / run_transform / run_distort,
// :122-233) needs only an include swap.  The reference's Matrix is an Eigen
// row-major double matrix; Eigen is not required here: Matrix below is a
// row-major double buffer with the same indexing (m(i, j), rows(), cols(),
// data(), row pointers).  All arithmetic runs on the B200 through libadg.so.
//
// Link:  -I include  -L paper_1609_05388_b200 -ladg  (plus -Wl,-rpath).
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <numeric>
#include <string_view>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "adg.h"

namespace adagio {

// ----------------------------------------------------- point_cloud.hpp
class Matrix {
 public:
  Matrix() = default;
  Matrix(int64_t rows, int64_t cols) { resize(rows, cols); }
  void resize(int64_t rows, int64_t cols) {
    rows_ = rows;
    cols_ = cols;
    data_.assign(static_cast<size_t>(rows * cols), 0.0);
  }
  int64_t rows() const { return rows_; }
  int64_t cols() const { return cols_; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  double& operator()(int64_t i, int64_t j) { return data_[static_cast<size_t>(i * cols_ + j)]; }
  double operator()(int64_t i, int64_t j) const { return data_[static_cast<size_t>(i * cols_ + j)]; }
  const double* row(int64_t i) const { return data() + i * cols_; }
  double* row(int64_t i) { return data() + i * cols_; }
  bool operator==(const Matrix& o) const {
    return rows_ == o.rows_ && cols_ == o.cols_ && data_ == o.data_;
  }

 private:
  int64_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

using Vector = std::vector<double>;

struct PointCloud {
  Matrix data;  // n x d
  std::optional<std::vector<int>> labels;
  int64_t n() const { return data.rows(); }
  int64_t d() const { return data.cols(); }
  bool has_labels() const { return labels.has_value(); }
};

// ------------------------------------------------------------ errors.hpp
struct IoError : std::runtime_error {
  explicit IoError(const std::string& what) : std::runtime_error(what) {}
};
struct NumericError : std::runtime_error {
  explicit NumericError(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
inline void check(adg_status st) {
  if (st == ADG_OK) return;
  const std::string msg = adg_last_error();
  switch (st) {
    case ADG_EINVAL: throw std::invalid_argument(msg);
    case ADG_ENUMERIC: throw NumericError(msg);
    case ADG_EIO: throw IoError(msg);
    default: throw std::runtime_error(msg);
  }
}
inline adg_ctx* ctx() {
  struct Holder {
    adg_ctx* c = nullptr;
    ~Holder() {
      if (c) adg_ctx_destroy(c);
    }
  };
  static thread_local Holder h;
  if (!h.c) check(adg_ctx_create(0, &h.c));
  return h.c;
}
}  // namespace detail

// --------------------------------------------------------------- rng.hpp
inline std::uint64_t derive_seed(std::uint64_t seed, const std::string& purpose) {
  return adg_derive_seed(seed, purpose.c_str());
}

// ---------------------------------------------------------------- jl.hpp
struct JlMatrix {
  Matrix entries;  // k x d
  std::uint64_t seed = 0;
  int64_t k() const { return entries.rows(); }
  int64_t d() const { return entries.cols(); }
};

inline JlMatrix sample_jl(int64_t k, int64_t d, std::uint64_t seed) {
  if (k < 1 || d < 1) throw std::invalid_argument("sample_jl: k and d must be >= 1");
  JlMatrix m;
  m.seed = seed;
  m.entries.resize(k, d);
  detail::check(adg_sample_jl(detail::ctx(), k, d, seed, m.entries.data()));
  return m;
}

inline std::size_t jl_dimension(std::size_t n_points, double epsilon, double gamma) {
  int64_t out = 0;
  detail::check(adg_jl_dimension(static_cast<int64_t>(n_points), epsilon, gamma, &out));
  return static_cast<std::size_t>(out);
}

// ----------------------------------------------------------- dataset.hpp
struct CenteringInfo {
  Vector mean;
};

inline std::pair<PointCloud, CenteringInfo> center(const PointCloud& cloud) {
  PointCloud out;
  out.data.resize(cloud.n(), cloud.d());
  out.labels = cloud.labels;
  CenteringInfo info;
  info.mean.resize(static_cast<size_t>(cloud.d()));
  detail::check(adg_center(detail::ctx(), cloud.data.data(), ADG_F64, cloud.n(), cloud.d(),
                           info.mean.data(), out.data.data()));
  return {std::move(out), std::move(info)};
}

// ---------------------------------------------------------- spectral.hpp
struct OrthonormalBasis {
  Matrix rows;  // s x d
  int64_t s() const { return rows.rows(); }
  int64_t d() const { return rows.cols(); }
};
struct SpectralSummary {
  Vector singular_values;
  bool approximate = false;
};

inline std::pair<OrthonormalBasis, SpectralSummary> exact_top_svd(const PointCloud& cloud,
                                                                  int64_t s) {
  const int64_t r = std::min(cloud.n(), cloud.d());
  OrthonormalBasis b;
  b.rows.resize(s > 0 ? s : 0, cloud.d());
  SpectralSummary sm;
  sm.singular_values.resize(static_cast<size_t>(r > 0 ? r : 0));
  detail::check(adg_exact_top_svd(detail::ctx(), cloud.data.data(), ADG_F64, cloud.n(), cloud.d(),
                                  s, b.rows.data(), sm.singular_values.data(), r));
  return {std::move(b), std::move(sm)};
}

inline std::pair<OrthonormalBasis, SpectralSummary> randomized_top_svd(
    const PointCloud& cloud, int64_t s, int64_t oversampling = 10, int power_iters = 2,
    std::uint64_t seed = 0) {
  OrthonormalBasis b;
  b.rows.resize(s > 0 ? s : 0, cloud.d());
  SpectralSummary sm;
  sm.singular_values.resize(static_cast<size_t>(s > 0 ? s : 0));
  sm.approximate = true;
  detail::check(adg_randomized_top_svd(detail::ctx(), cloud.data.data(), ADG_F64, cloud.n(),
                                       cloud.d(), s, oversampling, power_iters, seed,
                                       b.rows.data(), sm.singular_values.data()));
  return {std::move(b), std::move(sm)};
}

// ------------------------------------------------------------- embed.hpp
enum class SpectralBackend : std::uint8_t { exact = 0, randomized = 1 };

struct AdagioModel {
  Vector mean;
  OrthonormalBasis basis;
  JlMatrix sketch;
  std::uint64_t seed = 0;
  SpectralBackend backend = SpectralBackend::exact;
  int64_t d() const { return sketch.d(); }
  int64_t s() const { return basis.s(); }
  int64_t k() const { return sketch.k(); }
  int64_t target_dim() const { return s() + k(); }
};

inline AdagioModel fit_with_split(const PointCloud& cloud, int64_t s, int64_t k,
                                  SpectralBackend backend, std::uint64_t seed) {
  AdagioModel m;
  m.mean.resize(static_cast<size_t>(cloud.d()));
  m.basis.rows.resize(s > 0 ? s : 0, cloud.d());
  m.sketch.entries.resize(k > 0 ? k : 0, cloud.d());
  detail::check(adg_fit_with_split(detail::ctx(), cloud.data.data(), ADG_F64, cloud.n(), cloud.d(),
                                   s, k, static_cast<adg_backend>(backend), seed, m.mean.data(),
                                   m.basis.rows.data(), m.sketch.entries.data()));
  m.sketch.seed = derive_seed(seed, "jl");
  m.seed = seed;
  m.backend = backend;
  return m;
}

inline AdagioModel fit(const PointCloud& cloud, int64_t target_dim, SpectralBackend backend,
                       std::uint64_t seed) {
  if (target_dim < 2 || target_dim > cloud.d())
    throw std::invalid_argument("fit: target_dim = " + std::to_string(target_dim) +
                                " outside [2, " + std::to_string(cloud.d()) + "]");
  if (cloud.n() < 2) throw std::invalid_argument("fit: need at least 2 points");
  return fit_with_split(cloud, target_dim / 2, target_dim - target_dim / 2, backend, seed);
}

inline PointCloud transform_all(const AdagioModel& model, const PointCloud& cloud) {
  if (cloud.d() != model.d())
    throw std::invalid_argument("transform_all: cloud dimension " + std::to_string(cloud.d()) +
                                ", model expects " + std::to_string(model.d()));
  PointCloud out;
  out.data.resize(cloud.n(), model.target_dim());
  out.labels = cloud.labels;
  detail::check(adg_transform_all(detail::ctx(), model.mean.data(),
                                  model.s() ? model.basis.rows.data() : nullptr, model.s(),
                                  model.sketch.entries.data(), model.k(), model.d(),
                                  cloud.data.data(), ADG_F64, cloud.n(), out.data.data(), ADG_F64));
  return out;
}

inline Vector transform(const AdagioModel& model, const Vector& w) {
  if (static_cast<int64_t>(w.size()) != model.d())
    throw std::invalid_argument("transform: vector has dimension " + std::to_string(w.size()) +
                                ", model expects " + std::to_string(model.d()));
  PointCloud one;
  one.data.resize(1, model.d());
  std::memcpy(one.data.data(), w.data(), sizeof(double) * w.size());
  const PointCloud y = transform_all(model, one);
  return Vector(y.data.data(), y.data.data() + y.data.cols());
}

// ADG1 model file, bit-exact (proj/include/adagio/embed.hpp:49-54,
// proj/src/embed.cpp:183-239): "ADG1", u32 version 1, u32 d, s, k, u8
// backend, u64 seed, then mean, P, S as little-endian IEEE doubles.
namespace detail {
inline void put_u32(std::ostream& o, std::uint32_t v) {
  unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16),
                        (unsigned char)(v >> 24)};
  o.write(reinterpret_cast<const char*>(b), 4);
}
inline void put_u64(std::ostream& o, std::uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(v >> (8 * i));
  o.write(reinterpret_cast<const char*>(b), 8);
}
inline std::uint64_t get_u64(std::istream& in, const std::string& path) {
  unsigned char b[8];
  in.read(reinterpret_cast<char*>(b), 8);
  if (!in) throw IoError("model: truncated file " + path);
  std::uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= std::uint64_t{b[i]} << (8 * i);
  return v;
}
inline std::uint32_t get_u32(std::istream& in, const std::string& path) {
  unsigned char b[4];
  in.read(reinterpret_cast<char*>(b), 4);
  if (!in) throw IoError("model: truncated file " + path);
  return std::uint32_t{b[0]} | (std::uint32_t{b[1]} << 8) | (std::uint32_t{b[2]} << 16) |
         (std::uint32_t{b[3]} << 24);
}
inline void put_doubles(std::ostream& o, const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    std::uint64_t bits;
    std::memcpy(&bits, &v[i], 8);
    put_u64(o, bits);
  }
}
inline void get_doubles(std::istream& in, double* v, size_t n, const std::string& path) {
  for (size_t i = 0; i < n; ++i) {
    const std::uint64_t bits = get_u64(in, path);
    std::memcpy(&v[i], &bits, 8);
  }
}
}  // namespace detail

inline void save_model(const AdagioModel& model, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("model: cannot write " + path);
  out.write("ADG1", 4);
  detail::put_u32(out, 1);
  detail::put_u32(out, (std::uint32_t)model.d());
  detail::put_u32(out, (std::uint32_t)model.s());
  detail::put_u32(out, (std::uint32_t)model.k());
  const unsigned char tag = static_cast<unsigned char>(model.backend);
  out.write(reinterpret_cast<const char*>(&tag), 1);
  detail::put_u64(out, model.seed);
  detail::put_doubles(out, model.mean.data(), (size_t)model.d());
  detail::put_doubles(out, model.basis.rows.data(), (size_t)(model.s() * model.d()));
  detail::put_doubles(out, model.sketch.entries.data(), (size_t)(model.k() * model.d()));
  if (!out) throw IoError("model: write failed for " + path);
}

inline AdagioModel load_model(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("model: cannot open " + path);
  char magic[4];
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "ADG1", 4) != 0) throw IoError("model: bad magic in " + path);
  const std::uint32_t version = detail::get_u32(in, path);
  if (version != 1)
    throw IoError("model: unsupported version " + std::to_string(version) + " in " + path);
  const std::uint32_t d = detail::get_u32(in, path), s = detail::get_u32(in, path),
                      k = detail::get_u32(in, path);
  if (d == 0 || k == 0) throw IoError("model: invalid dimensions in " + path);
  unsigned char tag = 0;
  in.read(reinterpret_cast<char*>(&tag), 1);
  if (!in) throw IoError("model: truncated file " + path);
  if (tag > 1) throw IoError("model: unknown backend tag in " + path);
  AdagioModel m;
  m.backend = static_cast<SpectralBackend>(tag);
  m.seed = detail::get_u64(in, path);
  m.mean.resize(d);
  detail::get_doubles(in, m.mean.data(), d, path);
  m.basis.rows.resize(s, d);
  detail::get_doubles(in, m.basis.rows.data(), (size_t)s * d, path);
  m.sketch.entries.resize(k, d);
  detail::get_doubles(in, m.sketch.entries.data(), (size_t)k * d, path);
  m.sketch.seed = derive_seed(m.seed, "jl");
  return m;
}

// -------------------------------------------------------- distortion.hpp
struct PairSampling {
  bool all_pairs = true;
  std::uint64_t m = 0;
  std::uint64_t seed = 0;
  static PairSampling all() { return {}; }
  static PairSampling sample(std::uint64_t m, std::uint64_t seed) { return {false, m, seed}; }
};

struct DistortionReport {
  double max_distortion = 0.0;
  double mean_distortion = 0.0;
  std::vector<std::uint64_t> histogram;
  int hist_bins = 0;
  double hist_max = 0.0;
  std::uint64_t n_pairs_evaluated = 0;
  std::uint64_t n_zero_distance_pairs = 0;
  bool sampled = false;
  std::optional<std::uint64_t> sample_seed;
  // extension: lowest (i, j) attaining the maximum (absent if nothing evaluated)
  std::optional<std::pair<std::uint64_t, std::uint64_t>> argmax;
};

namespace detail {
inline DistortionReport to_report(const adg_report& rep, std::vector<std::uint64_t> hist);
}  // namespace detail

inline DistortionReport evaluate(const PointCloud& original, const PointCloud& embedded,
                                 const PairSampling& mode, int hist_bins = 50,
                                 double hist_max = 1.0, std::uint64_t pairs_per_block = 16384) {
  adg_pair_sampling ps{mode.all_pairs ? 1 : 0, 0, mode.m, mode.seed};
  adg_report rep{};
  std::vector<std::uint64_t> hist(static_cast<size_t>(hist_bins > 0 ? hist_bins : 0) + 1);
  detail::check(adg_evaluate(detail::ctx(), original.data.data(), ADG_F64, original.n(),
                             original.d(), embedded.data.data(), ADG_F64, embedded.n(),
                             embedded.d(), &ps, hist_bins, hist_max, pairs_per_block,
                             ADG_ENGINE_AUTO, &rep, hist.data()));
  return detail::to_report(rep, std::move(hist));
}

// Extension: run_distort's --model flow (adagio_main.cpp:192-224) in one call,
// evaluate(original, transform_all(model, original), ...) with the original
// staged to the GPU once and the embedding kept there (adg_distort_model).
inline DistortionReport distort_with_model(const AdagioModel& model, const PointCloud& original,
                                           const PairSampling& mode, int hist_bins = 50,
                                           double hist_max = 1.0) {
  if (original.d() != model.d())
    throw std::invalid_argument("transform_all: cloud dimension " + std::to_string(original.d()) +
                                ", model expects " + std::to_string(model.d()));
  adg_pair_sampling ps{mode.all_pairs ? 1 : 0, 0, mode.m, mode.seed};
  adg_report rep{};
  std::vector<std::uint64_t> hist(static_cast<size_t>(hist_bins > 0 ? hist_bins : 0) + 1);
  detail::check(adg_distort_model(detail::ctx(), model.mean.data(),
                                  model.s() ? model.basis.rows.data() : nullptr, model.s(),
                                  model.sketch.entries.data(), model.k(), model.d(),
                                  original.data.data(), ADG_F64, original.n(), &ps, hist_bins,
                                  hist_max, ADG_ENGINE_AUTO, &rep, hist.data(), nullptr, ADG_F64));
  return detail::to_report(rep, std::move(hist));
}

namespace detail {
inline DistortionReport to_report(const adg_report& rep, std::vector<std::uint64_t> hist) {
  DistortionReport r;
  r.max_distortion = rep.max_distortion;
  r.mean_distortion = rep.mean_distortion;
  r.histogram = std::move(hist);
  r.hist_bins = rep.hist_bins;
  r.hist_max = rep.hist_max;
  r.n_pairs_evaluated = rep.n_pairs_evaluated;
  r.n_zero_distance_pairs = rep.n_zero_distance_pairs;
  r.sampled = rep.sampled != 0;
  if (r.sampled) r.sample_seed = rep.sample_seed;
  if (rep.argmax_i != UINT64_MAX) r.argmax = std::make_pair(rep.argmax_i, rep.argmax_j);
  return r;
}
}  // namespace detail

inline double max_distortion(const PointCloud& original, const PointCloud& embedded) {
  return evaluate(original, embedded, PairSampling::all()).max_distortion;
}

inline double pair_distortion(const Vector& x, const Vector& y, const Vector& fx,
                              const Vector& fy) {
  double out = 0.0;
  detail::check(adg_pair_distortion(detail::ctx(), x.data(), y.data(), (int64_t)x.size(),
                                    fx.data(), fy.data(), (int64_t)fx.size(), &out));
  return out;
}

namespace detail {
inline adg_report to_c(const DistortionReport& r) {
  adg_report c{};
  c.max_distortion = r.max_distortion;
  c.mean_distortion = r.mean_distortion;
  c.n_pairs_evaluated = r.n_pairs_evaluated;
  c.n_zero_distance_pairs = r.n_zero_distance_pairs;
  c.argmax_i = r.argmax ? r.argmax->first : UINT64_MAX;
  c.argmax_j = r.argmax ? r.argmax->second : UINT64_MAX;
  c.hist_bins = r.hist_bins;
  c.hist_max = r.hist_max;
  c.sampled = r.sampled;
  c.sample_seed = r.sample_seed.value_or(0);
  return c;
}
}  // namespace detail

// JSON text with the keys of proj/docs/schemas/distort.schema.json (the
// reference returns an nlohmann::json; callers here get its dump()).
inline std::string report_to_json(const DistortionReport& r) {
  const adg_report c = detail::to_c(r);
  std::string s(adg_report_to_json(&c, r.histogram.data(), nullptr, 0), '\0');
  adg_report_to_json(&c, r.histogram.data(), s.data(), s.size() + 1);
  return s;
}

inline std::string histogram_csv(const DistortionReport& r) {
  const adg_report c = detail::to_c(r);
  std::string s(adg_histogram_csv(&c, r.histogram.data(), nullptr, 0), '\0');
  adg_histogram_csv(&c, r.histogram.data(), s.data(), s.size() + 1);
  return s;
}

// ------------------------------------------------- proj/include/adagio/sweep.hpp
enum class Method { adagio_exact, adagio_randomized, pca, jl, external };

inline const char* method_name(Method method) { return adg_method_name(static_cast<int32_t>(method)); }

inline Method method_from_name(const std::string& name) {
  int32_t m = 0;
  detail::check(adg_method_from_name(name.c_str(), &m));
  return static_cast<Method>(m);
}

struct SweepRow {
  Method method = Method::pca;
  int64_t target_dim = 0;
  std::uint64_t seed = 0;
  double max_distortion = 0.0;
  double fit_seconds = 0.0;
  double eval_seconds = 0.0;
};

inline std::vector<SweepRow> tradeoff(const PointCloud& cloud, const std::vector<int64_t>& dims,
                                      const std::vector<Method>& methods,
                                      const std::vector<std::uint64_t>& seeds,
                                      const PairSampling& eval_mode = PairSampling::all(),
                                      const Matrix* external_map = nullptr) {
  std::vector<int32_t> ms;
  for (const Method m : methods) ms.push_back(static_cast<int32_t>(m));
  int64_t count = 0;
  for (const Method m : methods)
    count += (m == Method::external ? 1 : (int64_t)dims.size()) * (int64_t)seeds.size();
  std::vector<adg_sweep_row> rows((size_t)std::max<int64_t>(count, 1));
  adg_pair_sampling ps{eval_mode.all_pairs ? 1 : 0, 0, eval_mode.m, eval_mode.seed};
  int64_t written = 0;
  detail::check(adg_tradeoff(detail::ctx(), cloud.data.data(), ADG_F64, cloud.n(), cloud.d(),
                             dims.data(), (int64_t)dims.size(), ms.data(), (int64_t)ms.size(),
                             seeds.data(), (int64_t)seeds.size(), &ps,
                             external_map ? external_map->data() : nullptr,
                             external_map ? external_map->rows() : 0,
                             external_map ? external_map->cols() : 0, rows.data(),
                             (int64_t)rows.size(), &written));
  std::vector<SweepRow> out;
  for (int64_t i = 0; i < written; ++i)
    out.push_back({static_cast<Method>(rows[i].method), rows[i].target_dim, rows[i].seed,
                   rows[i].max_distortion, rows[i].fit_seconds, rows[i].eval_seconds});
  return out;
}

struct MinDimResult {
  int64_t target_dim = 0;
  double achieved_distortion = 0.0;
  bool achieved = false;
  bool monotone = true;
};

inline MinDimResult min_dim_for_distortion(const PointCloud& cloud, Method method, double delta,
                                           std::uint64_t seed, int64_t r_min, int64_t r_max) {
  adg_min_dim_result r{};
  detail::check(adg_min_dim_for_distortion(detail::ctx(), cloud.data.data(), ADG_F64, cloud.n(),
                                           cloud.d(), static_cast<int32_t>(method), delta, seed,
                                           r_min, r_max, &r));
  return {r.target_dim, r.achieved_distortion, r.achieved != 0, r.monotone != 0};
}

inline std::string sweep_csv(const std::vector<SweepRow>& rows) {
  std::vector<adg_sweep_row> c;
  for (const SweepRow& r : rows)
    c.push_back({static_cast<int32_t>(r.method), 0, r.target_dim, r.seed, r.max_distortion,
                 r.fit_seconds, r.eval_seconds});
  std::string s(adg_sweep_csv(c.data(), (int64_t)c.size(), nullptr, 0), '\0');
  adg_sweep_csv(c.data(), (int64_t)c.size(), s.data(), s.size() + 1);
  return s;
}

// ------------------------------------------ proj/include/adagio/dataset.hpp I/O
// Host-side data formats around the path (proj/src/dataset.cpp:20-207, same
// syntax, bit-exact round trips and the same IoError messages).
namespace detail {
inline std::string_view csv_trim(std::string_view s) {
  while (!s.empty() && (s.front() == ' ' || s.front() == '\t')) s.remove_prefix(1);
  while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
  return s;
}
inline void csv_split(std::string_view line, std::vector<std::string_view>& out) {
  out.clear();
  std::size_t start = 0;
  for (std::size_t i = 0; i <= line.size(); ++i)
    if (i == line.size() || line[i] == ',') {
      out.push_back(csv_trim(line.substr(start, i - start)));
      start = i + 1;
    }
}
inline double csv_field(std::string_view f, std::size_t row, std::size_t col) {
  double v = 0.0;
  const auto r = std::from_chars(f.data(), f.data() + f.size(), v);
  if (r.ec != std::errc{} || r.ptr != f.data() + f.size() || f.empty())
    throw IoError("csv: non-numeric field '" + std::string(f) + "' at row " + std::to_string(row) +
                  ", column " + std::to_string(col));
  if (!std::isfinite(v))
    throw IoError("csv: non-finite value at row " + std::to_string(row) + ", column " +
                  std::to_string(col));
  return v;
}
inline std::uint32_t read_be_u32(std::istream& in, const std::string& path) {
  unsigned char b[4];
  in.read(reinterpret_cast<char*>(b), 4);
  if (!in) throw IoError("idx: truncated header in " + path);
  return (std::uint32_t{b[0]} << 24) | (std::uint32_t{b[1]} << 16) | (std::uint32_t{b[2]} << 8) |
         std::uint32_t{b[3]};
}
}  // namespace detail

// proj/src/dataset.cpp:72-121
inline PointCloud load_csv(const std::string& path, bool has_header = false,
                           std::optional<int> label_column = std::nullopt) {
  std::ifstream in(path);
  if (!in) throw IoError("csv: cannot open " + path);
  std::vector<std::vector<double>> rows;
  std::vector<int> labels;
  std::vector<std::string_view> fields;
  std::string line;
  std::size_t line_no = 0, expected = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (has_header && line_no == 1) continue;
    if (detail::csv_trim(line).empty()) continue;
    detail::csv_split(line, fields);
    if (expected == 0) {
      expected = fields.size();
      if (label_column && (*label_column < 0 || static_cast<std::size_t>(*label_column) >= expected))
        throw IoError("csv: label column " + std::to_string(*label_column) + " out of range for " +
                      std::to_string(expected) + " columns");
    } else if (fields.size() != expected) {
      throw IoError("csv: row " + std::to_string(line_no) + " has " + std::to_string(fields.size()) +
                    " fields, expected " + std::to_string(expected));
    }
    std::vector<double> row;
    row.reserve(expected);
    for (std::size_t c = 0; c < fields.size(); ++c) {
      const double v = detail::csv_field(fields[c], line_no, c + 1);
      if (label_column && static_cast<std::size_t>(*label_column) == c) {
        if (v < 0.0 || v != std::floor(v) || v > static_cast<double>(std::numeric_limits<int>::max()))
          throw IoError("csv: label must be a non-negative integer at row " + std::to_string(line_no) +
                        ", column " + std::to_string(c + 1));
        labels.push_back(static_cast<int>(v));
      } else {
        row.push_back(v);
      }
    }
    rows.push_back(std::move(row));
  }
  if (rows.empty()) throw IoError("csv: no data rows in " + path);
  if (rows.front().empty()) throw IoError("csv: no feature columns in " + path);
  PointCloud cloud;
  cloud.data.resize((int64_t)rows.size(), (int64_t)rows.front().size());
  for (int64_t i = 0; i < cloud.n(); ++i)
    for (int64_t j = 0; j < cloud.d(); ++j) cloud.data(i, j) = rows[(size_t)i][(size_t)j];
  if (label_column) cloud.labels = std::move(labels);
  return cloud;
}

// proj/src/dataset.cpp:123-141 (%.17g: reloading is bit-exact)
inline std::string csv_string(const PointCloud& cloud, bool with_labels = true) {
  char buf[40];
  std::string out;
  const bool emit_labels = with_labels && cloud.has_labels();
  for (int64_t i = 0; i < cloud.n(); ++i) {
    for (int64_t j = 0; j < cloud.d(); ++j) {
      if (j > 0) out += ',';
      std::snprintf(buf, sizeof(buf), "%.17g", cloud.data(i, j));
      out += buf;
    }
    if (emit_labels) {
      out += ',';
      out += std::to_string((*cloud.labels)[(size_t)i]);
    }
    out += '\n';
  }
  return out;
}

inline void save_csv(const PointCloud& cloud, const std::string& path, bool with_labels = true) {
  std::ofstream out(path);
  if (!out) throw IoError("csv: cannot write " + path);
  out << csv_string(cloud, with_labels);
  if (!out) throw IoError("csv: write failed for " + path);
}

// proj/src/dataset.cpp:150-207 (MNIST IDX: big-endian header, u8 pixels)
inline PointCloud load_idx(const std::string& images_path,
                           const std::optional<std::string>& labels_path = std::nullopt) {
  std::ifstream in(images_path, std::ios::binary);
  if (!in) throw IoError("idx: cannot open " + images_path);
  if (detail::read_be_u32(in, images_path) != 0x00000803u)
    throw IoError("idx: wrong magic in " + images_path + " (expected 0x00000803)");
  const std::uint32_t count = detail::read_be_u32(in, images_path);
  const std::uint32_t rows = detail::read_be_u32(in, images_path);
  const std::uint32_t cols = detail::read_be_u32(in, images_path);
  if (count == 0 || rows == 0 || cols == 0) throw IoError("idx: empty image file " + images_path);
  const std::size_t pixels = std::size_t{count} * rows * cols;
  std::vector<unsigned char> bytes(pixels);
  in.read(reinterpret_cast<char*>(bytes.data()), (std::streamsize)pixels);
  if ((std::size_t)in.gcount() != pixels) throw IoError("idx: truncated image payload in " + images_path);
  PointCloud cloud;
  cloud.data.resize(count, (int64_t)rows * cols);
  for (std::size_t t = 0; t < pixels; ++t) cloud.data.data()[t] = (double)bytes[t];
  if (labels_path) {
    std::ifstream lin(*labels_path, std::ios::binary);
    if (!lin) throw IoError("idx: cannot open " + *labels_path);
    if (detail::read_be_u32(lin, *labels_path) != 0x00000801u)
      throw IoError("idx: wrong magic in " + *labels_path + " (expected 0x00000801)");
    const std::uint32_t lcount = detail::read_be_u32(lin, *labels_path);
    if (lcount != count)
      throw IoError("idx: image/label count mismatch (" + std::to_string(count) + " images, " +
                    std::to_string(lcount) + " labels)");
    std::vector<unsigned char> lb(lcount);
    lin.read(reinterpret_cast<char*>(lb.data()), (std::streamsize)lcount);
    if ((std::size_t)lin.gcount() != lcount) throw IoError("idx: truncated label payload in " + *labels_path);
    cloud.labels = std::vector<int>(lb.begin(), lb.end());
  }
  return cloud;
}

// proj/src/dataset.cpp:218-245 (partial Fisher-Yates with SeededRng.below)
inline PointCloud sample_points(const PointCloud& cloud, int64_t m, std::uint64_t seed) {
  if (m < 1 || m > cloud.n())
    throw std::invalid_argument("sample_points: m = " + std::to_string(m) + " outside [1, " +
                                std::to_string(cloud.n()) + "]");
  std::vector<int64_t> index((size_t)cloud.n());
  std::iota(index.begin(), index.end(), int64_t{0});
  std::uint64_t state = seed;
  auto next = [&state]() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  auto below = [&next](std::uint64_t bound) {
    const std::uint64_t limit = bound * ((~std::uint64_t{0}) / bound);
    std::uint64_t v = next();
    while (v >= limit) v = next();
    return v % bound;
  };
  for (int64_t i = 0; i < m; ++i) {
    const int64_t off = (int64_t)below((std::uint64_t)(cloud.n() - i));
    std::swap(index[(size_t)i], index[(size_t)(i + off)]);
  }
  PointCloud out;
  out.data.resize(m, cloud.d());
  std::vector<int> labels;
  for (int64_t i = 0; i < m; ++i) {
    const int64_t src = index[(size_t)i];
    for (int64_t j = 0; j < cloud.d(); ++j) out.data(i, j) = cloud.data(src, j);
    if (cloud.has_labels()) labels.push_back((*cloud.labels)[(size_t)src]);
  }
  if (cloud.has_labels()) out.labels = std::move(labels);
  return out;
}

}  // namespace adagio
