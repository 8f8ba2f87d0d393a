// adagio_b200.hpp -- header-only C++17 facade with the reference's API.
//
// Reproduces the names, structs, defaults and exception types of the
// reference headers proj/include/adagio/{point_cloud,errors,rng,parallel,jl,
// spectral,embed,distortion,dataset}.hpp on top of the C ABI in adg.h; the
// shims include/adagio/*.hpp carry the reference's header names, so a caller
// such as proj/tools/adagio_main.cpp (run_fit / run_transform / run_distort,
// :122-233) compiles with only the include path swapped
// (tests/test_dropin_compile.py).  With Eigen on the include path, Matrix /
// Vector are the reference's Eigen types (point_cloud.hpp:12-13); without it,
// Matrix is a row-major double buffer with the subset of that interface the
// callers use.  With nlohmann's json.hpp on the include path, report_to_json
// returns the reference's nlohmann::json (distortion.hpp:60).  All arithmetic
// runs on the B200 through libadg.so.
//
// Link:  -I include  -L paper_1609_05388_b200 -ladg  (plus -Wl,-rpath).
#pragma once

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <limits>
#include <numeric>
#include <string_view>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "adg.h"

#if __has_include(<Eigen/Core>) && !defined(ADAGIO_B200_NO_EIGEN)
#include <Eigen/Core>
#define ADAGIO_B200_EIGEN 1
#else
namespace Eigen {
using Index = std::ptrdiff_t;  // what the reference's callers cast sizes to
}  // namespace Eigen
#endif
#if __has_include(<json.hpp>) && !defined(ADAGIO_B200_NO_JSON)
#include <json.hpp>
#define ADAGIO_B200_JSON 1
#endif

namespace adagio {

// ----------------------------------------------------- point_cloud.hpp
#ifdef ADAGIO_B200_EIGEN
using Matrix = Eigen::Matrix<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>;
using Vector = Eigen::VectorXd;
#else
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
  // the first k columns (Eigen's leftCols, as adagio_main.cpp:209 uses it)
  Matrix leftCols(int64_t k) const {
    Matrix m(rows_, k);
    for (int64_t i = 0; i < rows_; ++i) std::copy(row(i), row(i) + k, m.row(i));
    return m;
  }

 private:
  int64_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

using Vector = std::vector<double>;
#endif

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
  std::memcpy(one.data.data(), w.data(), sizeof(double) * (size_t)w.size());
  const PointCloud y = transform_all(model, one);
  Vector out;
  out.resize(y.data.cols());
  std::copy(y.data.data(), y.data.data() + y.data.cols(), out.data());
  return out;
}

// ADG1 model files (proj/include/adagio/embed.hpp:49-54; byte layout of
// proj/src/embed.cpp:183-239, the interchange format):
//   offset 0  "ADG1"          4 bytes
//          4  version = 1     u32 LE
//          8  d, s, k         3 x u32 LE
//         20  backend tag     u8 (0 exact, 1 randomized)
//         21  seed            u64 LE
//         29  mean[d], P[s*d], S[k*d]   IEEE-754 doubles, LE
// The file is assembled in memory and written (or read whole and parsed) in
// one go; ModelBytes bounds-checks every read.
namespace detail {
static_assert(sizeof(double) == 8 && std::numeric_limits<double>::is_iec559, "IEEE doubles");

struct ModelBytes {
  std::vector<unsigned char> buf;
  std::size_t at = 0;
  std::string path;
  template <typename T>
  void append(T v) {  // little-endian, whatever the host order
    unsigned char b[sizeof(T)];
    std::uint64_t bits = 0;
    std::memcpy(&bits, &v, sizeof(T));
    for (std::size_t i = 0; i < sizeof(T); ++i) b[i] = (unsigned char)(bits >> (8 * i));
    buf.insert(buf.end(), b, b + sizeof(T));
  }
  template <typename T>
  T take() {
    if (buf.size() - at < sizeof(T)) throw IoError("model: truncated file " + path);
    std::uint64_t bits = 0;
    for (std::size_t i = 0; i < sizeof(T); ++i) bits |= std::uint64_t{buf[at + i]} << (8 * i);
    at += sizeof(T);
    T v;
    std::memcpy(&v, &bits, sizeof(T));
    return v;
  }
  void append_all(const double* v, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i) append(v[i]);
  }
  void take_all(double* v, std::size_t n) {
    for (std::size_t i = 0; i < n; ++i) v[i] = take<double>();
  }
};
}  // namespace detail

inline void save_model(const AdagioModel& model, const std::string& path) {
  detail::ModelBytes f;
  for (char c : {'A', 'D', 'G', '1'}) f.append((unsigned char)c);
  for (std::uint32_t v : {1u, (std::uint32_t)model.d(), (std::uint32_t)model.s(),
                          (std::uint32_t)model.k()})
    f.append(v);
  f.append(static_cast<unsigned char>(model.backend));
  f.append(model.seed);
  f.append_all(model.mean.data(), (size_t)model.d());
  f.append_all(model.basis.rows.data(), (size_t)(model.s() * model.d()));
  f.append_all(model.sketch.entries.data(), (size_t)(model.k() * model.d()));
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("model: cannot write " + path);
  out.write(reinterpret_cast<const char*>(f.buf.data()), (std::streamsize)f.buf.size());
  if (!out) throw IoError("model: write failed for " + path);
}

inline AdagioModel load_model(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("model: cannot open " + path);
  detail::ModelBytes f;
  f.path = path;
  f.buf.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
  if (f.buf.size() < 4 || std::memcmp(f.buf.data(), "ADG1", 4) != 0)
    throw IoError("model: bad magic in " + path);
  f.at = 4;
  const auto version = f.take<std::uint32_t>();
  if (version != 1)
    throw IoError("model: unsupported version " + std::to_string(version) + " in " + path);
  const auto d = f.take<std::uint32_t>(), s = f.take<std::uint32_t>(), k = f.take<std::uint32_t>();
  if (d == 0 || k == 0) throw IoError("model: invalid dimensions in " + path);
  const auto tag = f.take<unsigned char>();
  if (tag > 1) throw IoError("model: unknown backend tag in " + path);
  AdagioModel m;
  m.backend = static_cast<SpectralBackend>(tag);
  m.seed = f.take<std::uint64_t>();
  m.mean.resize(d);
  f.take_all(m.mean.data(), d);
  m.basis.rows.resize(s, d);
  f.take_all(m.basis.rows.data(), (size_t)s * d);
  m.sketch.entries.resize(k, d);
  f.take_all(m.sketch.entries.data(), (size_t)k * d);
  m.sketch.seed = derive_seed(m.seed, "jl");
  return m;
}

// ----------------------------------------------------------- parallel.hpp
// proj/include/adagio/parallel.hpp:12-13.  The host-thread budget is kept for
// API compatibility (the CLI sets it from --threads / ADAGIO_THREADS); the
// work runs on the GPU.  Its GPU analogue: evaluate() shards all-pairs jobs
// over gpu_budget() GPUs of this process (set_gpu_budget, or ADAGIO_GPUS;
// default 1) with NCCL between them (adg_evaluate_multi) -- results are
// bit-identical for any budget, as the reference's are for any thread count.
namespace detail {
inline int& thread_budget_slot() {
  static int n = 0;
  return n;
}
inline int& gpu_budget_slot() {
  static int n = [] {
    const char* e = std::getenv("ADAGIO_GPUS");
    return e && std::atoi(e) > 0 ? std::atoi(e) : 1;
  }();
  return n;
}
}  // namespace detail
inline int thread_budget() {
  const int n = detail::thread_budget_slot();
  return n > 0 ? n : (int)std::max(1u, std::thread::hardware_concurrency());
}
inline void set_thread_budget(int n) { detail::thread_budget_slot() = n; }
inline int gpu_budget() { return detail::gpu_budget_slot(); }
inline void set_gpu_budget(int n) { detail::gpu_budget_slot() = n > 0 ? n : 1; }

// Extension: the evaluate() engine (adg_engine).  AUTO (default): the
// reference's fp64 block evaluator up to n = 4096 and for sampled pairs, the
// tensor-core SCREEN above (counts, max, argmax exact; mean within 1e-4;
// histogram exact away from bin edges).  EXACT gives the reference's numbers
// at any n (fp64 direct differences for every pair: C3 in ~0.3 s);
// SCREEN_EXACT_HIST its histogram bin for bin.  set_engine(), or ADAGIO_ENGINE
// = auto | exact | screen | screen_exact_hist.
namespace detail {
inline adg_engine& engine_slot() {
  static adg_engine e = [] {
    const char* v = std::getenv("ADAGIO_ENGINE");
    const std::string s = v ? v : "auto";
    if (s == "exact") return ADG_ENGINE_EXACT;
    if (s == "screen") return ADG_ENGINE_SCREEN;
    if (s == "screen_exact_hist") return ADG_ENGINE_SCREEN_EXACT_HIST;
    if (s != "auto") throw std::invalid_argument("ADAGIO_ENGINE: unknown engine '" + s + "'");
    return ADG_ENGINE_AUTO;
  }();
  return e;
}
}  // namespace detail
inline adg_engine engine() { return detail::engine_slot(); }
inline void set_engine(adg_engine e) { detail::engine_slot() = e; }

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
  if (gpu_budget() > 1) {
    std::vector<std::int32_t> devs((size_t)gpu_budget());
    std::iota(devs.begin(), devs.end(), 0);
    detail::check(adg_evaluate_multi((std::int32_t)devs.size(), devs.data(), original.data.data(),
                                     ADG_F64, original.n(), original.d(), embedded.data.data(),
                                     ADG_F64, embedded.n(), embedded.d(), &ps, hist_bins, hist_max,
                                     engine(), &rep, hist.data()));
  } else {
    detail::check(adg_evaluate(detail::ctx(), original.data.data(), ADG_F64, original.n(),
                               original.d(), embedded.data.data(), ADG_F64, embedded.n(),
                               embedded.d(), &ps, hist_bins, hist_max, pairs_per_block,
                               engine(), &rep, hist.data()));
  }
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
                                  hist_max, engine(), &rep, hist.data(), nullptr, ADG_F64));
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

// The keys of proj/docs/schemas/distort.schema.json: report_json_text is the
// document as text; report_to_json is the reference's nlohmann::json when
// json.hpp is on the include path, else that text.
inline std::string report_json_text(const DistortionReport& r) {
  const adg_report c = detail::to_c(r);
  std::string s(adg_report_to_json(&c, r.histogram.data(), nullptr, 0), '\0');
  adg_report_to_json(&c, r.histogram.data(), s.data(), s.size() + 1);
  return s;
}
#ifdef ADAGIO_B200_JSON
inline nlohmann::json report_to_json(const DistortionReport& r) {
  return nlohmann::json::parse(report_json_text(r));
}
#else
inline std::string report_to_json(const DistortionReport& r) { return report_json_text(r); }
#endif

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
// Host-side data formats around the path (the formats and IoError messages
// of proj/src/dataset.cpp:20-245, so files and failures interchange with the
// reference).  Each reader loads the whole file and scans it in memory.
namespace detail {
inline std::string slurp(const std::string& path, std::ios::openmode mode, const char* what) {
  std::ifstream in(path, mode);
  if (!in) throw IoError(std::string(what) + ": cannot open " + path);
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

// One CSV record: fields between commas, blanks and tabs ignored at both
// ends of a field (and a trailing CR at the end of the record).
struct CsvRecord {
  std::vector<std::string_view> fields;
  bool blank = true;
  void parse(std::string_view rec) {
    fields.clear();
    blank = true;
    const char* p = rec.data();
    const char* const end = p + rec.size();
    while (true) {
      const char* f0 = p;
      while (p < end && *p != ',') ++p;
      const char* f1 = p;
      while (f0 < f1 && (*f0 == ' ' || *f0 == '\t')) ++f0;
      while (f1 > f0 && (f1[-1] == ' ' || f1[-1] == '\t' || f1[-1] == '\r')) --f1;
      fields.emplace_back(f0, (std::size_t)(f1 - f0));
      if (f1 > f0 || p < end) blank = false;
      if (p == end) break;
      ++p;  // past the comma
    }
  }
};

inline double csv_number(std::string_view f, std::size_t row, std::size_t col) {
  double v = 0.0;
  const char* const e = f.data() + f.size();
  const auto r = std::from_chars(f.data(), e, v);
  const std::string where = " at row " + std::to_string(row) + ", column " + std::to_string(col);
  if (f.empty() || r.ec != std::errc{} || r.ptr != e)
    throw IoError("csv: non-numeric field '" + std::string(f) + "'" + where);
  if (!std::isfinite(v)) throw IoError("csv: non-finite value" + where);
  return v;
}

inline std::uint32_t be32(const std::string& b, std::size_t at) {
  return (std::uint32_t{(unsigned char)b[at]} << 24) | (std::uint32_t{(unsigned char)b[at + 1]} << 16) |
         (std::uint32_t{(unsigned char)b[at + 2]} << 8) | std::uint32_t{(unsigned char)b[at + 3]};
}

// rng.hpp SeededRng (splitmix64 stream, rejection-sampled below())
struct SplitMix {
  std::uint64_t s;
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  std::uint64_t below(std::uint64_t bound) {
    const std::uint64_t limit = bound * (~std::uint64_t{0} / bound);
    for (;;)
      if (const std::uint64_t v = next(); v < limit) return v % bound;
  }
};
}  // namespace detail

// proj/src/dataset.cpp:72-121 (load_csv)
inline PointCloud load_csv(const std::string& path, bool has_header = false,
                           std::optional<int> label_column = std::nullopt) {
  const std::string text = detail::slurp(path, std::ios::in, "csv");
  std::vector<double> values;
  std::vector<int> labels;
  std::size_t width = 0, nrows = 0, line_no = 0;
  detail::CsvRecord rec;
  for (std::size_t pos = 0; pos < text.size();) {
    std::size_t nl = text.find('\n', pos);
    if (nl == std::string::npos) nl = text.size();
    const std::string_view line(text.data() + pos, nl - pos);
    pos = nl + 1;
    ++line_no;
    if (has_header && line_no == 1) continue;
    rec.parse(line);
    if (rec.blank) continue;
    const std::size_t nf = rec.fields.size();
    if (width == 0) {
      width = nf;
      if (label_column && (*label_column < 0 || (std::size_t)*label_column >= width))
        throw IoError("csv: label column " + std::to_string(*label_column) + " out of range for " +
                      std::to_string(width) + " columns");
    } else if (nf != width) {
      throw IoError("csv: row " + std::to_string(line_no) + " has " + std::to_string(nf) +
                    " fields, expected " + std::to_string(width));
    }
    for (std::size_t c = 0; c < nf; ++c) {
      const double v = detail::csv_number(rec.fields[c], line_no, c + 1);
      if (!label_column || (std::size_t)*label_column != c) {
        values.push_back(v);
        continue;
      }
      const bool integral = v >= 0.0 && v == std::floor(v) &&
                            v <= (double)std::numeric_limits<int>::max();
      if (!integral)
        throw IoError("csv: label must be a non-negative integer at row " + std::to_string(line_no) +
                      ", column " + std::to_string(c + 1));
      labels.push_back((int)v);
    }
    ++nrows;
  }
  if (nrows == 0) throw IoError("csv: no data rows in " + path);
  const std::size_t d = width - (label_column ? 1 : 0);
  if (d == 0) throw IoError("csv: no feature columns in " + path);
  PointCloud cloud;
  cloud.data.resize((int64_t)nrows, (int64_t)d);
  std::copy(values.begin(), values.end(), cloud.data.data());
  if (label_column) cloud.labels = std::move(labels);
  return cloud;
}

// proj/src/dataset.cpp:123-141 (%.17g: a reload is bit-exact)
inline std::string csv_string(const PointCloud& cloud, bool with_labels = true) {
  const bool emit_labels = with_labels && cloud.has_labels();
  std::string out;
  out.reserve((size_t)(cloud.n() * (cloud.d() * 24 + 8)));
  char num[40];
  for (int64_t i = 0; i < cloud.n(); ++i) {
    const double* row = cloud.data.data() + i * cloud.d();
    for (int64_t j = 0; j < cloud.d(); ++j) {
      const int len = std::snprintf(num, sizeof(num), "%.17g", row[j]);
      if (j) out.push_back(',');
      out.append(num, (size_t)len);
    }
    if (emit_labels) out.append(",").append(std::to_string((*cloud.labels)[(size_t)i]));
    out.push_back('\n');
  }
  return out;
}

inline void save_csv(const PointCloud& cloud, const std::string& path, bool with_labels = true) {
  const std::string text = csv_string(cloud, with_labels);
  std::ofstream out(path);
  if (!out) throw IoError("csv: cannot write " + path);
  out.write(text.data(), (std::streamsize)text.size());
  if (!out) throw IoError("csv: write failed for " + path);
}

// proj/src/dataset.cpp:150-207 (MNIST IDX: big-endian u32 header, u8 payload)
inline PointCloud load_idx(const std::string& images_path,
                           const std::optional<std::string>& labels_path = std::nullopt) {
  const std::string img = detail::slurp(images_path, std::ios::binary, "idx");
  if (img.size() < 4) throw IoError("idx: truncated header in " + images_path);
  if (detail::be32(img, 0) != 0x00000803u)
    throw IoError("idx: wrong magic in " + images_path + " (expected 0x00000803)");
  if (img.size() < 16) throw IoError("idx: truncated header in " + images_path);
  const std::uint32_t count = detail::be32(img, 4), h = detail::be32(img, 8), w = detail::be32(img, 12);
  if (count == 0 || h == 0 || w == 0) throw IoError("idx: empty image file " + images_path);
  const std::size_t pixels = std::size_t{count} * h * w;
  if (img.size() - 16 < pixels) throw IoError("idx: truncated image payload in " + images_path);
  PointCloud cloud;
  cloud.data.resize(count, (int64_t)h * w);
  const unsigned char* px = reinterpret_cast<const unsigned char*>(img.data()) + 16;
  std::transform(px, px + pixels, cloud.data.data(), [](unsigned char b) { return (double)b; });
  if (labels_path) {
    const std::string lab = detail::slurp(*labels_path, std::ios::binary, "idx");
    if (lab.size() < 4) throw IoError("idx: truncated header in " + *labels_path);
    if (detail::be32(lab, 0) != 0x00000801u)
      throw IoError("idx: wrong magic in " + *labels_path + " (expected 0x00000801)");
    if (lab.size() < 8) throw IoError("idx: truncated header in " + *labels_path);
    const std::uint32_t lcount = detail::be32(lab, 4);
    if (lcount != count)
      throw IoError("idx: image/label count mismatch (" + std::to_string(count) + " images, " +
                    std::to_string(lcount) + " labels)");
    if (lab.size() - 8 < lcount) throw IoError("idx: truncated label payload in " + *labels_path);
    const unsigned char* lb = reinterpret_cast<const unsigned char*>(lab.data()) + 8;
    cloud.labels = std::vector<int>(lb, lb + lcount);
  }
  return cloud;
}

// proj/src/dataset.cpp:218-245 (sample_points): the first m slots of a
// partial Fisher-Yates shuffle of the row indices, SeededRng(seed).below.
inline PointCloud sample_points(const PointCloud& cloud, int64_t m, std::uint64_t seed) {
  if (m < 1 || m > cloud.n())
    throw std::invalid_argument("sample_points: m = " + std::to_string(m) + " outside [1, " +
                                std::to_string(cloud.n()) + "]");
  std::vector<int64_t> perm((size_t)cloud.n());
  std::iota(perm.begin(), perm.end(), int64_t{0});
  detail::SplitMix rng{seed};
  for (int64_t i = 0; i < m; ++i)
    std::swap(perm[(size_t)i], perm[(size_t)(i + (int64_t)rng.below((std::uint64_t)(cloud.n() - i)))]);
  PointCloud out;
  out.data.resize(m, cloud.d());
  if (cloud.has_labels()) out.labels = std::vector<int>((size_t)m);
  for (int64_t i = 0; i < m; ++i) {
    const int64_t src = perm[(size_t)i];
    const double* from = cloud.data.data() + src * cloud.d();
    std::copy(from, from + cloud.d(), out.data.data() + i * cloud.d());
    if (cloud.has_labels()) (*out.labels)[(size_t)i] = (*cloud.labels)[(size_t)src];
  }
  return out;
}

}  // namespace adagio
