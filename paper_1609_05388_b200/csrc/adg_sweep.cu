// adg_sweep.cu -- dimension-distortion sweeps (proj/src/sweep.cpp) on the GPU.
//
// The reference centres the cloud once, caches one exact SVD and, per
// (method, dim, seed) cell, multiplies the centred data by the cell's map
// and runs the full distortion evaluator.  Here the cloud never leaves HBM
// and is never copied: each cell's map W (r x d: P for pca, S for jl, M for
// external, [P; S(I - P^T P)] for adagio) goes through the fused transform
// Y = (X - mean) W^T, and the cell is scored by the max-only evaluator on
// (X, Y) -- distortion is shift-invariant, so scoring against X instead of
// the centred copy only removes the centring's rounding.  The exact basis is
// computed once, at the largest rank the sweep can ask for, and prefixed per
// cell (proj/src/sweep.cpp:27-52 caches the full-rank SVD the same way).
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "adg_eval.cuh"
#include "adg_spectral.cuh"

namespace adg {
namespace {

using Clock = std::chrono::steady_clock;

double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

const char* const kMethodNames[] = {"adagio_exact", "adagio_randomized", "pca", "jl", "external"};

// proj/src/sweep.cpp:27-52 (ExactBasisCache), computed at `rank` rows.
struct BasisCache {
  adg_ctx* ctx;
  const void* X;
  adg_dtype dt;
  int64_t n, d, rank;
  const double* mean;
  DevBuf<double> rows;
  bool ready = false;
  int64_t max_rank() const { return std::min(n, d); }
  const double* get() {
    if (!ready && rank > 0) {
      rows.alloc((size_t)(rank * d), ctx->stream);
      spectral_exact(ctx, X, dt, n, d, mean, rank, rows.ptr, nullptr, 0, "exact_top_svd");
      ready = true;
    }
    return rows.ptr;
  }
};

struct Sweep {
  adg_ctx* ctx;
  const void* X;
  adg_dtype dt;
  int64_t n, d;
  DevBuf<double> mean;
  std::unique_ptr<BasisCache> cache;
  const double* external = nullptr;  // device
  int64_t ext_rows = 0;

  Sweep(adg_ctx* c, const void* x, adg_dtype t, int64_t n_, int64_t d_, int64_t cache_rank)
      : ctx(c), X(x), dt(t), n(n_), d(d_), mean((size_t)d_, c->stream) {
    column_means(ctx, X, dt, n, d, mean.ptr);
    cache.reset(new BasisCache{ctx, X, dt, n, d, cache_rank, mean.ptr, {}, false});
  }

  // proj/src/sweep.cpp:60-137 (embed_cell) + the cell's max distortion.
  // upper != nullptr: row->max_distortion is a lower bound L and *upper an
  // upper bound U of the cell's maximum (see max_distortion_device)
  void cell(int32_t method, int64_t r, uint64_t seed, const adg_pair_sampling* mode,
            adg_sweep_row* row, double* upper = nullptr) {
    const auto t0 = Clock::now();
    int64_t s = 0, k = 0;
    const double* P = nullptr;
    const double* S = nullptr;
    DevBuf<double> sketch, fitted;
    switch (method) {
      case ADG_METHOD_PCA:
        // components beyond the usable rank carry zero variance (sweep.cpp:69-71)
        s = std::min(r, cache->max_rank());
        P = cache->get();
        break;
      case ADG_METHOD_JL:
        k = r;
        sketch.alloc((size_t)(k * d), ctx->stream);
        sample_jl_device(ctx, k, d, derive_seed(seed, "jl"), sketch.ptr);
        S = sketch.ptr;
        break;
      case ADG_METHOD_EXTERNAL:
        s = ext_rows;
        P = external;
        break;
      case ADG_METHOD_ADAGIO_EXACT:
      case ADG_METHOD_ADAGIO_RANDOMIZED: {
        s = r / 2;
        k = r - r / 2;
        sketch.alloc((size_t)(k * d), ctx->stream);
        sample_jl_device(ctx, k, d, derive_seed(seed, "jl"), sketch.ptr);
        S = sketch.ptr;
        if (s == 0) break;
        if (method == ADG_METHOD_ADAGIO_EXACT && s <= cache->max_rank()) {
          P = cache->get();  // zero-mean model on the centred cloud (sweep.cpp:104-118)
        } else {
          // fit_with_split(centered, s, k, backend, seed) (sweep.cpp:119-124)
          fitted.alloc((size_t)(s * d), ctx->stream);
          const int64_t mr = cache->max_rank();
          if (method == ADG_METHOD_ADAGIO_RANDOMIZED && s <= mr)
            spectral_randomized(ctx, X, dt, n, d, mean.ptr, s, std::min<int64_t>(10, mr - s), 2,
                                derive_seed(seed, "spectral"), fitted.ptr, nullptr);
          else
            spectral_exact(ctx, X, dt, n, d, mean.ptr, s, fitted.ptr, nullptr, 0, "exact_top_svd");
          P = fitted.ptr;
        }
        break;
      }
      default:
        fail(ADG_EINVAL, "sweep: unknown method");
    }
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
    row->fit_seconds = seconds_since(t0);
    const auto t1 = Clock::now();
    const int64_t rr = s + k;
    const adg_dtype ydt = dt == ADG_F64 ? ADG_F64 : ADG_F32;
    DevBuf<uint8_t> Y((size_t)(n * rr) * dtype_size(ydt), ctx->stream);
    {
      TransformPlan plan(ctx, mean.ptr, P, s, S, k, d, dt == ADG_F64);
      plan.run(X, dt, n, Y.ptr, ydt);
    }
    row->max_distortion = max_distortion_device(ctx, X, dt, n, d, Y.ptr, ydt, rr, mode, upper);
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
    row->eval_seconds = seconds_since(t1);
    row->method = method;
    row->reserved = 0;
    row->target_dim = method == ADG_METHOD_EXTERNAL ? ext_rows : r;
    row->seed = seed;
  }
};

void check_method(int32_t m) {
  if (m < 0 || m > ADG_METHOD_EXTERNAL) fail(ADG_EINVAL, "sweep: unknown method");
}

}  // namespace
}  // namespace adg

using namespace adg;

extern "C" {

const char* adg_method_name(int32_t method) {
  return (method >= 0 && method <= ADG_METHOD_EXTERNAL) ? kMethodNames[method] : "unknown";
}

// proj/src/sweep.cpp:152-159
adg_status adg_method_from_name(const char* name, int32_t* method_out) {
  return guard_call([&] {
    ADG_REQUIRE(name && method_out, "method_from_name: null argument");
    for (int32_t m = 0; m <= ADG_METHOD_EXTERNAL; ++m)
      if (std::strcmp(name, kMethodNames[m]) == 0) {
        *method_out = m;
        return;
      }
    fail(ADG_EINVAL, std::string("unknown method '") + name + "'");
  });
}

// proj/src/sweep.cpp:161-201
adg_status adg_tradeoff(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                        const int64_t* dims, int64_t n_dims, const int32_t* methods,
                        int64_t n_methods, const uint64_t* seeds, int64_t n_seeds,
                        const adg_pair_sampling* eval_mode, const double* external_map,
                        int64_t external_rows, int64_t external_cols, adg_sweep_row* rows_out,
                        int64_t rows_capacity, int64_t* rows_written) {
  return guard_call([&] {
    ADG_REQUIRE(ctx, "null adg_ctx");
    ADG_CUDA(cudaSetDevice(ctx->device));
    if (n_dims <= 0) fail(ADG_EINVAL, "tradeoff: dims must be non-empty");
    for (int64_t i = 0; i < n_dims; ++i)
      if (dims[i] < 1 || dims[i] > d)
        fail(ADG_EINVAL, "tradeoff: dim " + std::to_string(dims[i]) + " outside [1, " +
                             std::to_string(d) + "]");
    for (int64_t i = 0; i < n_methods; ++i) check_method(methods[i]);
    // rows: dims x seeds per method, one dim (the matrix's) for external
    int64_t total = 0;
    for (int64_t i = 0; i < n_methods; ++i)
      total += (methods[i] == ADG_METHOD_EXTERNAL ? 1 : n_dims) * std::max<int64_t>(n_seeds, 0);
    if (rows_written) *rows_written = total;
    ADG_REQUIRE(rows_capacity >= total, "tradeoff: rows_out too small");
    if (eval_mode && !eval_mode->all_pairs) {
      const uint64_t un = (uint64_t)std::max<int64_t>(n, 0);
      const uint64_t P = un * (un - (un ? 1 : 0)) / 2;
      if (eval_mode->m < 1 || eval_mode->m > P)
        fail(ADG_EINVAL, "evaluate: sample size " + std::to_string(eval_mode->m) +
                             " outside [1, " + std::to_string(P) + "]");
    }
    // the largest basis prefix any cell can use
    int64_t rank = 0;
    const int64_t mr = std::min(n, d);
    for (int64_t i = 0; i < n_methods; ++i)
      for (int64_t j = 0; j < n_dims; ++j) {
        if (methods[i] == ADG_METHOD_PCA) rank = std::max(rank, std::min(dims[j], mr));
        if (methods[i] == ADG_METHOD_ADAGIO_EXACT && dims[j] / 2 <= mr)
          rank = std::max(rank, dims[j] / 2);
      }
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    Sweep sw(ctx, x.dev, dtype, n, d, rank);
    std::unique_ptr<In> ext;
    int64_t out = 0;
    for (int64_t i = 0; i < n_methods; ++i) {
      const int32_t m = methods[i];
      if (m == ADG_METHOD_EXTERNAL) {
        if (!external_map) fail(ADG_EINVAL, "sweep: method external needs an embedding matrix");
        if (external_cols != d)
          fail(ADG_EINVAL, "sweep: external matrix has " + std::to_string(external_cols) +
                               " columns, cloud has " + std::to_string(d));
        ADG_REQUIRE(external_rows >= 1, "sweep: external matrix has no rows");
        if (!ext) ext.reset(new In(external_map, sizeof(double) * (size_t)(external_rows * d),
                                   ctx->stream));
        sw.external = ext->as<double>();
        sw.ext_rows = external_rows;
        for (int64_t q = 0; q < n_seeds; ++q)
          sw.cell(m, external_rows, seeds[q], eval_mode, &rows_out[out++]);
        continue;
      }
      for (int64_t j = 0; j < n_dims; ++j)
        for (int64_t q = 0; q < n_seeds; ++q) sw.cell(m, dims[j], seeds[q], eval_mode, &rows_out[out++]);
    }
  });
}

// proj/src/sweep.cpp:203-265
adg_status adg_min_dim_for_distortion(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n,
                                      int64_t d, int32_t method, double delta, uint64_t seed,
                                      int64_t r_min, int64_t r_max, adg_min_dim_result* out) {
  return guard_call([&] {
    ADG_REQUIRE(ctx && out, "min_dim_for_distortion: null argument");
    ADG_CUDA(cudaSetDevice(ctx->device));
    if (!(delta > 0.0 && delta < 1.0))
      fail(ADG_EINVAL, "min_dim_for_distortion: delta must lie in (0, 1)");
    if (r_min < 1 || r_min > r_max || r_max > d)
      fail(ADG_EINVAL, "min_dim_for_distortion: need 1 <= r_min <= r_max <= d");
    check_method(method);
    if (method == ADG_METHOD_EXTERNAL)
      fail(ADG_EINVAL, "min_dim_for_distortion: external maps have a fixed dimension");
    const int64_t mr = std::min(n, d);
    const int64_t rank = method == ADG_METHOD_PCA            ? std::min(r_max, mr)
                         : method == ADG_METHOD_ADAGIO_EXACT ? std::min(r_max / 2, mr)
                                                             : 0;
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    Sweep sw(ctx, x.dev, dtype, n, d, rank);
    // Every probe's maximum is first bracketed, L <= max <= U, by the screen
    // and the exact refine of its best row (the early exit of SURVEY 8f1): a
    // comparison with delta, or between neighbouring probes for the monotone
    // flag, refines the probe exactly only when the brackets cannot decide it.
    // The result is the reference's exactly (sweep.cpp:214-257).
    struct Bracket {
      double lo, hi;
      bool exact;
    };
    std::map<int64_t, Bracket> probed;
    auto bracket = [&](int64_t r) -> Bracket& {
      auto it = probed.find(r);
      if (it == probed.end()) {
        adg_sweep_row row;
        double up = 0.0;
        sw.cell(method, r, seed, nullptr, &row, &up);
        it = probed.emplace(r, Bracket{row.max_distortion, up, up <= row.max_distortion}).first;
      }
      return it->second;
    };
    int32_t refined = 0;
    auto exact = [&](int64_t r) {
      Bracket& b = bracket(r);
      if (!b.exact) {
        adg_sweep_row row;
        sw.cell(method, r, seed, nullptr, &row);
        b = Bracket{row.max_distortion, row.max_distortion, true};
        ++refined;
      }
      return b.lo;
    };
    auto within = [&](int64_t r) {  // max(r) <= delta
      const Bracket& b = bracket(r);
      if (b.hi <= delta) return true;
      if (b.lo > delta) return false;
      return exact(r) <= delta;
    };
    adg_min_dim_result res{};
    if (within(r_min)) {
      res.target_dim = r_min;
      res.achieved_distortion = exact(r_min);
      res.achieved = 1;
    } else {
      int64_t lo = r_min, hi = r_min;
      bool hi_ok = false;
      while (!hi_ok && hi < r_max) {
        lo = hi;
        hi = std::min<int64_t>(r_max, std::max<int64_t>(hi * 2, hi + 1));
        hi_ok = within(hi);
      }
      if (!hi_ok) {
        res.target_dim = r_max;
        res.achieved_distortion = exact(hi);
        res.achieved = 0;
      } else {
        while (hi - lo > 1) {
          const int64_t mid = lo + (hi - lo) / 2;
          if (within(mid))
            hi = mid;
          else
            lo = mid;
        }
        res.target_dim = hi;
        res.achieved_distortion = exact(hi);
        res.achieved = 1;
      }
    }
    // non-monotone iff some probe exceeds its predecessor (in r) by > 1e-12
    res.monotone = 1;
    int64_t prev_r = -1;
    for (auto& kv : probed) {
      if (prev_r >= 0) {
        const Bracket& a = probed.at(prev_r);
        const Bracket& b = kv.second;
        bool up;
        if (b.lo > a.hi + 1e-12)
          up = true;
        else if (b.hi <= a.lo + 1e-12)
          up = false;
        else
          up = exact(kv.first) > exact(prev_r) + 1e-12;
        if (up) res.monotone = 0;
      }
      prev_r = kv.first;
    }
    res.probes_refined = refined;
    res.probes = (int32_t)probed.size();
    *out = res;
  });
}

// proj/src/sweep.cpp:267-278
size_t adg_sweep_csv(const adg_sweep_row* rows, int64_t count, char* buf, size_t cap) {
  std::string s = "method,target_dim,seed,max_distortion,fit_seconds,eval_seconds\n";
  char line[200];
  for (int64_t i = 0; i < count; ++i) {
    std::snprintf(line, sizeof(line), "%s,%lld,%llu,%.17g,%.6f,%.6f\n",
                  adg_method_name(rows[i].method), (long long)rows[i].target_dim,
                  (unsigned long long)rows[i].seed, rows[i].max_distortion, rows[i].fit_seconds,
                  rows[i].eval_seconds);
    s += line;
  }
  if (buf && cap) {
    const size_t k = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return s.size();
}

}  // extern "C"
