// adg_api.cu -- the extern "C" boundary (include/adg.h).
//
// Validation and error messages follow the reference's functions one for one
// (file:line cited at each entry point); all arithmetic runs in the CUDA
// kernels of this library.  Host code here only validates, stages buffers,
// draws the sampled-pair indices (Floyd's algorithm is an inherently serial
// hash-set walk, proj/src/distortion.cpp:90-103) and formats output.
#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <string>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <memory>
#include <thread>
#include <unordered_set>

#include "adg_eval.cuh"
#include "adg_exact.cuh"
#include "adg_finalize.cuh"
#include "adg_screen.cuh"
#include "adg_spectral.cuh"

namespace adg {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

template <typename F>
static adg_status guard(F&& f) {
  try {
    f();
    return ADG_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return ADG_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return ADG_ECUDA;
  }
}

static void check_ctx(adg_ctx* ctx) {
  if (!ctx) fail(ADG_EINVAL, "null adg_ctx");
  ADG_CUDA(cudaSetDevice(ctx->device));
}



// proj/src/distortion.cpp:90-103 (Floyd), sorted.
static std::vector<uint64_t> sample_pair_indices(uint64_t total, uint64_t m, uint64_t seed) {
  std::unordered_set<uint64_t> chosen;
  chosen.reserve((size_t)m * 2);
  HostRng rng{seed};
  for (uint64_t t = total - m; t < total; ++t) {
    const uint64_t v = rng.below(t + 1);
    if (!chosen.insert(v).second) chosen.insert(t);
  }
  std::vector<uint64_t> idx(chosen.begin(), chosen.end());
  std::sort(idx.begin(), idx.end());
  return idx;
}

static void decode_pair_host(uint64_t p, uint64_t n, uint64_t& i, uint64_t& j) {
  const double nn = (double)n;
  double guess = std::floor((2.0 * nn - 1.0 - std::sqrt((2.0 * nn - 1.0) * (2.0 * nn - 1.0) - 8.0 * (double)p)) / 2.0);
  if (guess < 0.0) guess = 0.0;
  i = (uint64_t)guess;
  auto row_start = [n](uint64_t r) { return r * (2 * n - r - 1) / 2; };
  while (i > 0 && row_start(i) > p) --i;
  while (row_start(i + 1) <= p) ++i;
  j = i + 1 + (p - row_start(i));
}

static int bin_of_host(double value, int bins, double hist_max) {
  if (value >= hist_max) return bins;
  uint64_t b = (uint64_t)(value / hist_max * bins);
  if (b > (uint64_t)(bins - 1)) b = (uint64_t)(bins - 1);
  return (int)b;
}

struct NeuSum {
  double s = 0.0, c = 0.0;
  void add(double v) {
    const double t = s + v;
    if (std::fabs(s) >= std::fabs(v))
      c += (s - t) + v;
    else
      c += (v - t) + s;
    s = t;
  }
  double total() const { return s + c; }
};

}  // namespace adg

using namespace adg;

// ====================================================================== plan
struct adg_eval_plan {
  adg_ctx* ctx;
  cudaStream_t created_on = nullptr;  // its buffers' stream (the cache reuses it only there)
  std::unique_ptr<In> orig, emb;
  adg_dtype xd, yd;
  int64_t n, d, r;
  int bins;
  double hist_max;
  std::unique_ptr<ScreenOperands> ops;
  DevBuf<double> tile_sums;
  DevBuf<float> rows2;  // [row_max n | row_bound n]: one MAX all-reduce covers both
  float* row_max_ptr() { return rows2.ptr; }
  float* row_bound_ptr() { return rows2.ptr + n; }
  DevBuf<uint32_t> near_pairs;
  int64_t near_cap = 0;
  DevBuf<uint2> edge_pairs;  // pairs the screen could not bin (exact re-binning)
  int64_t edge_cap = 0;
  float edge_f = 0.f;  // edge band (ADG_ENGINE_SCREEN_EXACT_HIST: screen_edge_band(true))
  // set by a multi-GPU exchange: the best row and its exact refine (sharded
  // over the ranks) are already in the stage block for the finalize
  bool best_refined = false;
  // the collectives of the last exchange (valid until the finalize: a list
  // that did not fit the exchange's fixed-size gather is gathered again there)
  const adg_collectives* last_comm = nullptr;
  DevBuf<unsigned long long> own_near;  // this rank's near-coincident count, kept across the exchange
  // Everything the finalize reads back lives in one device block so a single
  // D2H copy (into the context's pinned staging) returns it:
  //   [near_count][tile total][best row][candidate count][edge slots][edge pairs]
  //   [hist bins+1][RowBest x refine chunks][candidate rows x n]
  static constexpr int64_t kHead = 6;
  DevBuf<unsigned long long> stage;
  int64_t refine_chunks = 0;
  unsigned long long* near_count() { return stage.ptr; }
  double* tile_total() { return reinterpret_cast<double*>(stage.ptr + 1); }
  int64_t* best_row() { return reinterpret_cast<int64_t*>(stage.ptr + 2); }
  unsigned long long* cand_count() { return stage.ptr + 3; }
  unsigned long long* edge_count() { return stage.ptr + 4; }  // slots reserved (list length)
  unsigned long long* edge_binned() { return stage.ptr + 5; }  // pairs binned exactly
  unsigned long long* hist() { return stage.ptr + kHead; }
  RowBest* best_row_refine() { return reinterpret_cast<RowBest*>(stage.ptr + kHead + 1 + bins); }
  int64_t* cand_rows() {
    return reinterpret_cast<int64_t*>(stage.ptr + kHead + 1 + bins + 3 * refine_chunks);
  }
};

static void plan_reset(adg_eval_plan* p) {
  p->best_refined = false;
  p->last_comm = nullptr;
  // near_count, tile total, best row, candidate count, edge count and histogram
  ADG_CUDA(cudaMemsetAsync(p->stage.ptr, 0, sizeof(unsigned long long) * (adg_eval_plan::kHead + 1 + p->bins),
                           p->ctx->stream));
  p->tile_sums.zero();
  p->rows2.zero();
}

// Capacity of the edge list: 1/128 of the pairs, within [2^20, 2^28] entries
// (C3: 14 M entries, 112 MB; the band puts ~0.1 % of C3's pairs there).  A
// run that needs more is redone in tile chunks by the finalize.
static int64_t edge_capacity(int64_t n) {
  const char* e = std::getenv("ADG_EDGE_CAP");  // testing aid: forces the chunked redo
  if (e && std::atoll(e) > 0) return std::atoll(e);
  const int64_t pairs = n * (n - 1) / 2;
  return std::max<int64_t>(1 << 20, std::min<int64_t>(pairs / 128, 1 << 28));
}

void* adg::pinned_stage(adg_ctx* ctx, size_t bytes) {
  if (bytes > ctx->pinned_bytes) {
    if (ctx->pinned) ADG_CUDA(cudaFreeHost(ctx->pinned));
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    const size_t sz = std::max<size_t>(bytes, 1 << 20);
    ADG_CUDA(cudaMallocHost(&ctx->pinned, sz));
    ctx->pinned_bytes = sz;
  }
  return ctx->pinned;
}

static adg_eval_plan* plan_create(adg_ctx* ctx, const void* orig, adg_dtype xd, int64_t n,
                                  int64_t d, const void* emb, adg_dtype yd, int64_t r, int bins,
                                  double hist_max,
                                  std::unique_ptr<ScreenOperands> ready_ops = nullptr) {
  auto p = std::make_unique<adg_eval_plan>();
  p->ctx = ctx;
  p->created_on = ctx->stream;
  p->xd = xd;
  p->yd = yd;
  p->n = n;
  p->d = d;
  p->r = r;
  p->bins = bins;
  p->hist_max = hist_max;
  p->orig = std::make_unique<In>(orig, (size_t)(n * d) * dtype_size(xd), ctx->stream);
  p->emb = std::make_unique<In>(emb, (size_t)(n * r) * dtype_size(yd), ctx->stream);
  p->ops = ready_ops ? std::move(ready_ops)
                     : std::make_unique<ScreenOperands>(ctx, p->orig->dev, xd, n, d, p->emb->dev, yd, r);
  p->refine_chunks = row_refine_chunks(n);
  static_assert(sizeof(RowBest) == 3 * sizeof(unsigned long long), "RowBest layout");
  p->stage.alloc((size_t)(adg_eval_plan::kHead + 1 + bins + 3 * p->refine_chunks + n), ctx->stream);
  p->tile_sums.alloc((size_t)(screen_tile_slots() * p->ops->num_tiles), ctx->stream);
  p->rows2.alloc((size_t)(2 * n), ctx->stream);
  p->near_cap = std::max<int64_t>(1 << 16, std::min<int64_t>(n * 16, 1 << 24));
  if (const char* e = std::getenv("ADG_NEAR_CAP"))  // testing aid: forces the chunked redo
    if (std::atoll(e) > 0) p->near_cap = std::atoll(e);
  p->near_pairs.alloc((size_t)(2 * p->near_cap), ctx->stream);
  p->edge_f = (float)screen_edge_band(false);
  p->edge_cap = edge_capacity(n);  // the list itself is allocated by the first exact-histogram run
  plan_reset(p.get());
  return p.release();
}

// The context's cached plan for device operands: same pointers, dtypes,
// shapes and histogram -> reset the partials and re-prepare the operands from
// the (possibly rewritten) data, skipping the allocations, tensor maps and
// tile-list setup.  Host inputs (staged copies) always get a fresh plan.
static bool plan_matches(const adg_eval_plan* p, const void* orig, adg_dtype xd, int64_t n, int64_t d,
                         const void* emb, adg_dtype yd, int64_t r, int bins, double hist_max) {
  return p && p->created_on == p->ctx->stream && p->orig->dev == orig && p->emb->dev == emb &&
         !p->orig->staged.ptr && !p->emb->staged.ptr &&
         p->xd == xd && p->yd == yd && p->n == n && p->d == d && p->r == r && p->bins == bins &&
         p->hist_max == hist_max;
}

static void plan_refresh(adg_eval_plan* p) {
  plan_reset(p);
  p->ops->refresh(p->orig->dev, p->xd, p->emb->dev, p->yd);
}

static adg_eval_plan* cached_plan(adg_ctx* ctx, const void* orig, adg_dtype xd, int64_t n, int64_t d,
                                  const void* emb, adg_dtype yd, int64_t r, int bins, double hist_max) {
  auto* cur = static_cast<adg_eval_plan*>(ctx->plan_cache);
  if (std::getenv("ADG_NO_PLAN_CACHE") == nullptr &&
      plan_matches(cur, orig, xd, n, d, emb, yd, r, bins, hist_max) && is_device_ptr(orig) &&
      is_device_ptr(emb)) {
    plan_refresh(cur);
    return cur;
  }
  delete cur;
  ctx->plan_cache = nullptr;
  adg_eval_plan* p = plan_create(ctx, orig, xd, n, d, emb, yd, r, bins, hist_max);
  if (!p->orig->staged.ptr && !p->emb->staged.ptr) ctx->plan_cache = p;
  return p;
}

static void release_plan(adg_ctx* ctx, adg_eval_plan* p) {
  if (p != ctx->plan_cache) delete p;
}

// Screen the tiles [t0, t1), then bin the edge pairs exactly into the same
// histogram (stream-ordered, no host round trip).  An edge list that
// overflowed marks the near-coincident count as overflowed too, so the
// finalize (after any multi-GPU exchange, which carries that count) redoes
// the histogram in tile chunks.
static void plan_screen(adg_eval_plan* p, int64_t t0, int64_t t1, bool max_only,
                        cudaStream_t stream = nullptr) {
  if (p->edge_f > 0.f && !max_only && !p->edge_pairs.ptr)
    p->edge_pairs.alloc((size_t)p->edge_cap, p->ctx->stream);  // (C4: up to 2 GB)
  ScreenPartials out{p->hist(), p->tile_sums.ptr, p->row_max_ptr(), p->row_bound_ptr(),
                     p->near_pairs.ptr, p->near_count(), (long long)p->near_cap,
                     p->edge_pairs.ptr, p->edge_count(), (long long)p->edge_cap, p->edge_f};
  run_screen(p->ctx, *p->ops, t0, t1, p->bins, p->hist_max, out, max_only, stream);
}

static void plan_edge_bin(adg_eval_plan* p) {
  if (p->edge_f > 0.f)
    run_edge_bin(p->ctx, p->orig->dev, p->xd, p->d, p->emb->dev, p->yd, p->r, p->edge_pairs.ptr,
                 p->edge_count(), p->edge_cap, p->bins, p->hist_max, p->hist(), p->edge_binned(),
                 p->near_count(), p->near_cap);
}

static void plan_run(adg_eval_plan* p, int64_t t0, int64_t t1, bool max_only = false) {
  plan_screen(p, t0, t1, max_only);
  if (!max_only && t1 > t0 && p->edge_f > 0.f)
    run_edge_bin(p->ctx, p->orig->dev, p->xd, p->d, p->emb->dev, p->yd, p->r, p->edge_pairs.ptr,
                 p->edge_count(), p->edge_cap, p->bins, p->hist_max, p->hist(), p->edge_binned(),
                 p->near_count(), p->near_cap);
}

// Exact engine over all pairs (also the overflow fallback of the screen).
static void evaluate_exact(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d,
                           const void* Y, adg_dtype yd, int64_t r, const uint64_t* sampled_dev,
                           uint64_t work, int bins, double hist_max, adg_report* rep,
                           uint64_t* hist_out) {
  DevBuf<unsigned long long> hist((size_t)bins + 1, ctx->stream);
  hist.zero();
  DevBuf<MergeOut> merged(1, ctx->stream);
  // ADG_EXACT_BLOCK: testing aid (the block engine at any size)
  if (!sampled_dev && n > 4096 && (size_t)(bins + 1) * sizeof(unsigned) <= 160 * 1024 &&
      !std::getenv("ADG_EXACT_BLOCK"))
    run_exact_tiled(ctx, X, xd, n, d, Y, yd, r, bins, hist_max, hist.ptr, merged.ptr);
  else
    run_exact(ctx, X, xd, n, d, Y, yd, r, sampled_dev, work, bins, hist_max, hist.ptr, merged.ptr);
  MergeOut m;
  ADG_CUDA(cudaMemcpyAsync(&m, merged.ptr, sizeof(m), cudaMemcpyDeviceToHost, ctx->stream));
  ADG_CUDA(cudaMemcpyAsync(hist_out, hist.ptr, sizeof(uint64_t) * (bins + 1),
                           cudaMemcpyDeviceToHost, ctx->stream));
  ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  rep->n_pairs_evaluated = m.evaluated;
  rep->n_zero_distance_pairs = m.zero;
  rep->max_distortion = m.evaluated ? m.max : 0.0;
  rep->mean_distortion = m.evaluated ? m.sum / (double)m.evaluated : 0.0;
  rep->argmax_i = rep->argmax_j = UINT64_MAX;
  if (m.evaluated && m.argp != UINT64_MAX) {
    if (sampled_dev) {
      // argp is the pair's linear index already (sampled list holds them)
    }
    decode_pair_host(m.argp, (uint64_t)n, rep->argmax_i, rep->argmax_j);
  }
  rep->engine = ADG_ENGINE_EXACT;
}

// near_count marker: some rank's list did not fit the exchange's first,
// fixed-size gather (the finalize gathers again, sized by the largest list)
constexpr unsigned long long kNearRegather = ~0ull - 1;
constexpr int64_t kNearBlock = 1024;  // pairs per rank in the first gather
extern "C" {
static unsigned long long near_regather(adg_eval_plan* p);  // (defined with the exchange)
}

// The near-coincident or edge list overflowed (this rank's or, after a
// multi-GPU exchange, any rank's): recompute the histogram and the
// near-coincident list over ALL tiles in chunks small enough for both lists
// (halving a chunk that still overflows), with the plan's buffers as per-chunk
// scratch.  The screen is deterministic per tile, so the tile sums and row
// maxima it rewrites are the values already there; the histogram is integer
// and the near pairs are sorted by the caller: the report is the one an
// unbounded list would give, for any GPU count.
static void plan_rechunk(adg_eval_plan* p, std::vector<uint64_t>& hist, std::vector<uint32_t>& pr,
                         std::vector<double>& hv, uint64_t& edges) {
  adg_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  std::fill(hist.begin(), hist.end(), 0);
  pr.clear();
  hv.clear();
  edges = 0;
  const int64_t T = p->ops->num_tiles;
  std::vector<std::pair<int64_t, int64_t>> todo;
  constexpr int64_t kChunks = 8;
  for (int64_t k = kChunks - 1; k >= 0; --k) todo.emplace_back(T * k / kChunks, T * (k + 1) / kChunks);
  const size_t head = sizeof(unsigned long long) * (size_t)(adg_eval_plan::kHead + 1 + p->bins);
  auto* hs = static_cast<unsigned long long*>(pinned_stage(ctx, head));
  while (!todo.empty()) {
    const auto [a, b] = todo.back();
    todo.pop_back();
    if (b <= a) continue;
    ADG_CUDA(cudaMemsetAsync(p->near_count(), 0, sizeof(unsigned long long), st));
    ADG_CUDA(cudaMemsetAsync(p->edge_count(), 0, sizeof(unsigned long long) * (size_t)(3 + p->bins), st));
    plan_run(p, a, b);
    ADG_CUDA(cudaMemcpyAsync(hs, p->stage.ptr, head, cudaMemcpyDeviceToHost, st));
    ADG_CUDA(cudaStreamSynchronize(st));
    const unsigned long long nc = hs[0], ec = hs[4], eb = hs[5];
    if ((int64_t)nc > p->near_cap || (int64_t)ec > p->edge_cap) {
      ADG_REQUIRE(b - a > 1, "evaluate: a single pair tile overflowed the exact-check lists");
      const int64_t mid = a + (b - a) / 2;
      todo.emplace_back(mid, b);
      todo.emplace_back(a, mid);
      continue;
    }
    for (int i = 0; i <= p->bins; ++i) hist[(size_t)i] += hs[adg_eval_plan::kHead + i];
    edges += eb;
    if (nc) {
      const int64_t c = (int64_t)nc;
      DevBuf<double> vals((size_t)c, st);
      run_pair_list(ctx, p->orig->dev, p->xd, p->d, p->emb->dev, p->yd, p->r, p->near_pairs.ptr, c,
                    vals.ptr);
      const size_t o = pr.size();
      pr.resize(o + (size_t)(2 * c));
      hv.resize(o / 2 + (size_t)c);
      ADG_CUDA(cudaMemcpyAsync(pr.data() + o, p->near_pairs.ptr, (size_t)(2 * c) * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, st));
      ADG_CUDA(cudaMemcpyAsync(hv.data() + o / 2, vals.ptr, (size_t)c * sizeof(double),
                               cudaMemcpyDeviceToHost, st));
      ADG_CUDA(cudaStreamSynchronize(st));
    }
  }
}

// upper != nullptr (max-only bounds): the candidate rows other than the best
// are not refined; *upper receives an upper bound of the maximum instead.
static void plan_finalize(adg_eval_plan* p, adg_report* rep, uint64_t* hist_out,
                          double* upper = nullptr) {
  adg_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const uint64_t n = (uint64_t)p->n;
  const uint64_t total_pairs = n * (n - 1) / 2;
  std::memset(rep, 0, sizeof(*rep));
  rep->hist_bins = p->bins;
  rep->hist_max = p->hist_max;
  rep->engine = p->edge_f > 0.f ? ADG_ENGINE_SCREEN_EXACT_HIST : ADG_ENGINE_SCREEN;
  rep->screen_error_bound = p->ops->eps;

  // Device chain with a single host round trip in the common case:
  //   ordered tile-sum; row with the largest screened value -> exact refine of
  //   that row -> lower bound L -> every row whose screened bound reaches L.
  const int64_t cpr = p->refine_chunks;
  constexpr int64_t kRowsPrefix = 4096;
  DevBuf<float> Lf(1, st);
  DevBuf<double> Ld(1, st);
  ADG_CUDA(cudaMemsetAsync(p->cand_count(), 0, sizeof(unsigned long long), st));
  ordered_sum(ctx, p->tile_sums.ptr, screen_tile_slots() * p->ops->num_tiles, p->tile_total());
  if (!p->best_refined) {  // (the multi-GPU exchange refined it, sharded)
    argmax_f32(ctx, p->row_max_ptr(), p->n, p->best_row());
    int64_t cpr_chk = 0;
    run_row_refine(ctx, p->orig->dev, p->xd, p->n, p->d, p->emb->dev, p->yd, p->r, p->best_row(), 1,
                   p->best_row_refine(), &cpr_chk);
  }
  row_lower_bound(ctx, reinterpret_cast<const double*>(p->best_row_refine()), cpr,
                  (int64_t)(sizeof(RowBest) / sizeof(double)), Lf.ptr, Ld.ptr);
  select_rows(ctx, p->row_bound_ptr(), p->n, Lf.ptr, p->cand_rows(), p->cand_count(), p->n);

  // one read-back of the whole head of the stage block (+ a prefix of rows)
  const int64_t nprefix = std::min<int64_t>(kRowsPrefix, p->n);
  constexpr int64_t H = adg_eval_plan::kHead;
  const size_t head = sizeof(unsigned long long) * (size_t)(H + 1 + p->bins + 3 * cpr + nprefix);
  auto* hs = static_cast<unsigned long long*>(pinned_stage(ctx, head + sizeof(unsigned long long)));
  ADG_CUDA(cudaMemcpyAsync(hs, p->stage.ptr, head, cudaMemcpyDeviceToHost, st));
  int* lo_flag_h = reinterpret_cast<int*>(reinterpret_cast<char*>(hs) + head);
  ADG_CUDA(cudaMemcpyAsync(lo_flag_h, p->ops->lo_flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  ADG_CUDA(cudaStreamSynchronize(st));
  ctx->last_orig_passes = (ctx->screen_forced3 || *lo_flag_h) ? 3 : 1;
  unsigned long long near_count = hs[0];
  if (near_count == kNearRegather) near_count = near_regather(p);
  p->last_comm = nullptr;
  double tile_total;
  int64_t brow;
  std::memcpy(&tile_total, hs + 1, sizeof(double));
  std::memcpy(&brow, hs + 2, sizeof(int64_t));
  const unsigned long long ncand_dev = hs[3];
  uint64_t edges = hs[5];
  std::vector<uint64_t> hist(hs + H, hs + H + 1 + p->bins);
  std::vector<RowBest> hb((size_t)cpr);
  std::memcpy(hb.data(), hs + H + 1 + p->bins, sizeof(RowBest) * hb.size());
  std::vector<int64_t> rows((size_t)nprefix);
  std::memcpy(rows.data(), hs + H + 1 + p->bins + 3 * cpr, sizeof(int64_t) * rows.size());
  // near-coincident pairs (i, j) and their exact values (-1: zero pair)
  std::vector<uint32_t> pr;
  std::vector<double> hv;
  if ((int64_t)near_count > p->near_cap) {
    plan_rechunk(p, hist, pr, hv, edges);
  } else if (near_count) {
    const int64_t c = (int64_t)near_count;
    DevBuf<double> vals((size_t)c, st);
    run_pair_list(ctx, p->orig->dev, p->xd, p->d, p->emb->dev, p->yd, p->r, p->near_pairs.ptr, c,
                  vals.ptr);
    pr.resize((size_t)(2 * c));
    hv.resize((size_t)c);
    ADG_CUDA(cudaMemcpyAsync(pr.data(), p->near_pairs.ptr, pr.size() * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, st));
    ADG_CUDA(cudaMemcpyAsync(hv.data(), vals.ptr, hv.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
    ADG_CUDA(cudaStreamSynchronize(st));
  }
  rep->edge_pairs = edges;

  double best = -1.0;
  int64_t bi = INT64_MAX, bj = INT64_MAX;
  auto consider = [&](double v, int64_t i, int64_t j) {
    if (v < 0.0) return;
    if (v > best || (v == best && (i < bi || (i == bi && j < bj)))) {
      best = v;
      bi = i;
      bj = j;
    }
  };
  auto refine_rows = [&](const std::vector<int64_t>& rows) {
    if (rows.empty()) return;
    DevBuf<int64_t> rows_dev(rows.size(), st);
    ADG_CUDA(cudaMemcpyAsync(rows_dev.ptr, rows.data(), rows.size() * sizeof(int64_t),
                             cudaMemcpyHostToDevice, st));
    int64_t cpr = 0;
    const int64_t cpr_est = row_refine_chunks(p->n);
    DevBuf<RowBest> outb((size_t)(rows.size() * cpr_est), st);
    run_row_refine(ctx, p->orig->dev, p->xd, p->n, p->d, p->emb->dev, p->yd, p->r, rows_dev.ptr,
                   (int64_t)rows.size(), outb.ptr, &cpr);
    std::vector<RowBest> hb(rows.size() * cpr);
    ADG_CUDA(cudaMemcpyAsync(hb.data(), outb.ptr, hb.size() * sizeof(RowBest),
                             cudaMemcpyDeviceToHost, st));
    ADG_CUDA(cudaStreamSynchronize(st));
    for (const RowBest& rb : hb) consider(rb.max, rb.i, rb.j);
  };
  // the row of the screened maximum was refined on the device already
  for (const RowBest& rb : hb) consider(rb.max, rb.i, rb.j);
  int64_t ncand = 0;
  if (brow >= 0) {
    const int64_t c = (int64_t)ncand_dev;
    if (c > (int64_t)rows.size()) {
      rows.resize((size_t)c);
      ADG_CUDA(cudaMemcpyAsync(rows.data(), p->cand_rows(), c * sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));
      ADG_CUDA(cudaStreamSynchronize(st));
    }
    rows.resize((size_t)c);
    std::sort(rows.begin(), rows.end());
    rows.erase(std::remove(rows.begin(), rows.end(), brow), rows.end());
    ncand = (int64_t)rows.size() + 1;
    if (!upper) {
      refine_rows(rows);  // every other row whose screened bound reaches L
    } else if (!rows.empty()) {
      // bounds only: the largest screened row bound (fp32; widened for its rounding)
      DevBuf<int64_t> ib(1, st);
      argmax_f32(ctx, p->row_bound_ptr(), p->n, ib.ptr);
      int64_t hi_row = 0;
      float ub = 0.f;
      ADG_CUDA(cudaMemcpyAsync(&hi_row, ib.ptr, sizeof(hi_row), cudaMemcpyDeviceToHost, st));
      ADG_CUDA(cudaStreamSynchronize(st));
      ADG_CUDA(cudaMemcpyAsync(&ub, p->row_bound_ptr() + hi_row, sizeof(ub), cudaMemcpyDeviceToHost, st));
      ADG_CUDA(cudaStreamSynchronize(st));
      *upper = (double)ub * (1.0 + 1e-6) + 1e-30;
    }
  }
  rep->candidate_rows = (int32_t)std::min<int64_t>(ncand, INT32_MAX);

  // 4. near-coincident pairs: exact zero rule, exact value into hist/sum/max
  uint64_t zero = 0;
  NeuSum near_sum;
  if (!hv.empty()) {
    const int64_t c = (int64_t)hv.size();
    std::vector<int64_t> order((size_t)c);
    for (int64_t k = 0; k < c; ++k) order[k] = k;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      return pr[2 * a] != pr[2 * b] ? pr[2 * a] < pr[2 * b] : pr[2 * a + 1] < pr[2 * b + 1];
    });
    for (int64_t k : order) {
      const double v = hv[k];
      if (v < 0.0) {
        ++zero;
        continue;
      }
      near_sum.add(v);
      hist[bin_of_host(v, p->bins, p->hist_max)]++;
      consider(v, pr[2 * k], pr[2 * k + 1]);
    }
  }

  NeuSum total;
  total.add(tile_total);
  total.add(near_sum.total());
  rep->n_zero_distance_pairs = zero;
  rep->n_pairs_evaluated = total_pairs - zero;
  rep->mean_distortion =
      rep->n_pairs_evaluated ? total.total() / (double)rep->n_pairs_evaluated : 0.0;
  rep->max_distortion = best >= 0.0 ? best : 0.0;
  if (upper) {
    // no other candidate row: the maximum is exact; else U covers the screened rows
    if (ncand <= 1 || *upper < rep->max_distortion) *upper = rep->max_distortion;
  }
  rep->argmax_i = best >= 0.0 ? (uint64_t)bi : UINT64_MAX;
  rep->argmax_j = best >= 0.0 ? (uint64_t)bj : UINT64_MAX;
  if (hist_out) std::memcpy(hist_out, hist.data(), hist.size() * sizeof(uint64_t));
}

// =================================================================== C ABI
extern "C" {

int adg_abi_version(void) { return ADG_ABI_VERSION; }
const char* adg_last_error(void) { return g_last_error.c_str(); }

adg_status adg_ctx_create(int device, adg_ctx** out) {
  return guard([&] {
    if (!out) fail(ADG_EINVAL, "adg_ctx_create: null out");
    int count = 0;
    ADG_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
      fail(ADG_ECUDA, "adg_ctx_create: no CUDA device " + std::to_string(device));
    ADG_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<adg_ctx>();
    c->device = device;
    ADG_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    int major = 0;
    ADG_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) fail(ADG_ECUDA, "libadg is built for sm_100a (B200); device is sm_" + std::to_string(major) + "x");
    ADG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    // Keep freed stream-ordered allocations in the device pool: the SCREEN
    // operands (hundreds of MB) are rebuilt per evaluation and must not go
    // back to the driver at every synchronisation.
    cudaMemPool_t pool;
    ADG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    ADG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    ADG_CUDA(cudaEventCreate(&c->ev_a));
    ADG_CUDA(cudaEventCreate(&c->ev_b));
    *out = c.release();
  });
}

adg_status adg_ctx_destroy(adg_ctx* ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    // the cached plan's buffers are freed on the context stream: before it goes
    delete static_cast<adg_eval_plan*>(ctx->plan_cache);
    ctx->plan_cache = nullptr;
    free_tile_list_cache(ctx);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    for (cudaStream_t s : ctx->phase_streams)
      if (s) cudaStreamDestroy(s);
    cudaEventDestroy(ctx->ev_a);
    cudaEventDestroy(ctx->ev_b);
    delete ctx;
  });
}

adg_status adg_ctx_set_stream(adg_ctx* ctx, void* stream) {
  return guard([&] {
    check_ctx(ctx);
    // the cached plan's buffers live on the old stream: free them there first
    delete static_cast<adg_eval_plan*>(ctx->plan_cache);
    ctx->plan_cache = nullptr;
    if (ctx->own_stream) ADG_CUDA(cudaStreamDestroy(ctx->stream));
    if (stream) {
      ctx->stream = (cudaStream_t)stream;
      ctx->own_stream = false;
    } else {
      ADG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
  });
}

adg_status adg_ctx_synchronize(adg_ctx* ctx) {
  return guard([&] {
    check_ctx(ctx);
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

uint64_t adg_derive_seed(uint64_t seed, const char* purpose) {
  return derive_seed(seed, purpose ? purpose : "");
}

// proj/src/jl.cpp:13-36
adg_status adg_sample_jl(adg_ctx* ctx, int64_t k, int64_t d, uint64_t seed, double* out) {
  return guard([&] {
    check_ctx(ctx);
    ADG_REQUIRE(k >= 1 && d >= 1, "sample_jl: k and d must be >= 1");
    Out o(out, sizeof(double) * (size_t)(k * d), ctx->stream);
    sample_jl_device(ctx, k, d, seed, o.as<double>());
    o.commit();
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// proj/src/jl.cpp:38-50
adg_status adg_jl_dimension(int64_t n_points, double epsilon, double gamma, int64_t* out) {
  return guard([&] {
    ADG_REQUIRE(n_points >= 2, "jl_dimension: need n_points >= 2");
    ADG_REQUIRE(epsilon > 0.0 && epsilon < 1.0, "jl_dimension: epsilon must lie in (0, 1)");
    ADG_REQUIRE(gamma > 0.0 && gamma < 1.0, "jl_dimension: gamma must lie in (0, 1)");
    const double n = (double)n_points;
    const double denom = epsilon * epsilon / 2.0 - epsilon * epsilon * epsilon / 3.0;
    const double k = 4.0 * std::log(n * n / gamma) / denom;
    *out = (int64_t)std::ceil(k);
  });
}

// proj/src/dataset.cpp:209-216
adg_status adg_center(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                      double* mean_out, void* centered_out) {
  return guard([&] {
    check_ctx(ctx);
    ADG_REQUIRE(n >= 1 && d >= 1, "center: empty cloud");
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    Out m(mean_out, sizeof(double) * (size_t)d, ctx->stream);
    column_means(ctx, x.dev, dtype, n, d, m.as<double>());
    if (centered_out) {
      Out c(centered_out, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
      center_into(ctx, x.dev, dtype, n, d, m.as<double>(), c.dev);
      c.commit();
      m.commit();
      ADG_CUDA(cudaStreamSynchronize(ctx->stream));
      return;
    }
    m.commit();
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adg_status adg_exact_top_svd(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                             int64_t s, double* basis_out, double* sigma_out, int64_t n_sigma) {
  return guard([&] {
    check_ctx(ctx);
    const int64_t max_rank = std::min(n, d);
    if (s < 1 || s > max_rank)
      fail(ADG_EINVAL, "exact_top_svd: s = " + std::to_string(s) + " outside [1, " +
                           std::to_string(max_rank) + "]");
    ADG_REQUIRE(n_sigma >= 0 && n_sigma <= max_rank, "exact_top_svd: n_sigma outside [0, min(n, d)]");
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    Out b(basis_out, sizeof(double) * (size_t)(s * d), ctx->stream);
    Out sg(sigma_out, sizeof(double) * (size_t)std::max<int64_t>(n_sigma, 0), ctx->stream);
    spectral_exact(ctx, x.dev, dtype, n, d, nullptr, s, b.as<double>(),
                   sigma_out ? sg.as<double>() : nullptr, sigma_out ? n_sigma : 0,
                   "exact_top_svd");
    b.commit();
    sg.commit();
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adg_status adg_randomized_top_svd(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n,
                                  int64_t d, int64_t s, int64_t oversampling, int power_iters,
                                  uint64_t seed, double* basis_out, double* sigma_out) {
  return guard([&] {
    check_ctx(ctx);
    const int64_t max_rank = std::min(n, d);
    if (s < 1 || oversampling < 0 || s + oversampling > max_rank)
      fail(ADG_EINVAL, "randomized_top_svd: need 1 <= s and s + oversampling <= " +
                           std::to_string(max_rank));
    ADG_REQUIRE(power_iters >= 0, "randomized_top_svd: power_iters must be >= 0");
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    Out b(basis_out, sizeof(double) * (size_t)(s * d), ctx->stream);
    Out sg(sigma_out, sizeof(double) * (size_t)s, ctx->stream);
    spectral_randomized(ctx, x.dev, dtype, n, d, nullptr, s, oversampling, power_iters, seed,
                        b.as<double>(), sigma_out ? sg.as<double>() : nullptr);
    b.commit();
    sg.commit();
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// proj/src/embed.cpp:115-141
adg_status adg_fit_with_split(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n,
                              int64_t d, int64_t s, int64_t k, adg_backend backend,
                              uint64_t seed, double* mean_out, double* basis_out,
                              double* sketch_out) {
  return guard([&] {
    NvtxRange nvtx_("adg_fit_with_split");
    check_ctx(ctx);
    if (s < 0 || s > d)
      fail(ADG_EINVAL, "fit_with_split: s = " + std::to_string(s) + " outside [0, " +
                           std::to_string(d) + "]");
    if (k < 1)
      fail(ADG_EINVAL,
           "fit_with_split: k must be >= 1 (for a pure principal projection use the sweep "
           "module's pca method)");
    if (n < 2) fail(ADG_EINVAL, "fit_with_split: need at least 2 points");
    if (s + k > d)
      std::cerr << "fit_with_split: warning: output dimension " << (s + k)
                << " exceeds ambient dimension " << d << "\n";
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    Out m(mean_out, sizeof(double) * (size_t)d, ctx->stream);
    Out b(basis_out, sizeof(double) * (size_t)(s * d), ctx->stream);
    Out sk(sketch_out, sizeof(double) * (size_t)(k * d), ctx->stream);
    column_means(ctx, x.dev, dtype, n, d, m.as<double>());
    if (s > 0) {
      const int64_t max_rank = std::min(n, d);
      if (s <= max_rank && backend == ADG_BACKEND_RANDOMIZED) {
        const int64_t over = std::min<int64_t>(10, max_rank - s);
        spectral_randomized(ctx, x.dev, dtype, n, d, m.as<double>(), s, over, 2,
                            derive_seed(seed, "spectral"), b.as<double>(), nullptr);
      } else {
        // s <= max_rank: exact_top_svd; s > max_rank: full eigenbasis (embed.cpp:46-55)
        spectral_exact(ctx, x.dev, dtype, n, d, m.as<double>(), s, b.as<double>(), nullptr, 0,
                       "exact_top_svd");
      }
    }
    sample_jl_device(ctx, k, d, derive_seed(seed, "jl"), sk.as<double>());
    m.commit();
    b.commit();
    sk.commit();
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ---------------------------------------------------------- sharded fit
// the fit's data-dependent work, split by rows.  Each
// rank sums its shard's columns (adg_column_sums), the sums are all-reduced
// and divided by the total row count (proj/src/dataset.cpp:211, colwise
// mean = sum / n), each rank forms the Gram of its centred shard
// (adg_gram), the d x d Grams are all-reduced, and every rank solves on the
// identical total (adg_fit_from_gram).  At one shard this is exactly
// adg_fit_with_split's arithmetic.
adg_status adg_column_sums(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                           double* sums_out) {
  return guard([&] {
    check_ctx(ctx);
    ADG_REQUIRE(n >= 0 && d >= 1, "column_sums: need n >= 0 and d >= 1");
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    Out o(sums_out, sizeof(double) * (size_t)d, ctx->stream);
    if (n == 0)
      ADG_CUDA(cudaMemsetAsync(o.dev, 0, sizeof(double) * (size_t)d, ctx->stream));
    else
      column_sums(ctx, x.dev, dtype, n, d, o.as<double>());
    o.commit();
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adg_status adg_gram(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                    const double* mean, adg_backend backend, double* gram_out) {
  return guard([&] {
    check_ctx(ctx);
    ADG_REQUIRE(n >= 0 && d >= 1, "gram: need n >= 0 and d >= 1");
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    In m(mean, sizeof(double) * (size_t)d, ctx->stream);
    Out g(gram_out, sizeof(double) * (size_t)(d * d), ctx->stream);
    if (n == 0) {
      ADG_CUDA(cudaMemsetAsync(g.dev, 0, sizeof(double) * (size_t)(d * d), ctx->stream));
    } else {
      require_finite(ctx, x.dev, dtype, n * d,
                     backend == ADG_BACKEND_RANDOMIZED ? "randomized_top_svd" : "exact_top_svd");
      gram_f64(ctx, x.dev, dtype, n, d, m.as<double>(), g.as<double>());
    }
    g.commit();
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adg_status adg_fit_from_gram(adg_ctx* ctx, const double* gram, int64_t n_total, int64_t d,
                             int64_t s, int64_t k, adg_backend backend, uint64_t seed,
                             double* basis_out, double* sketch_out) {
  return guard([&] {
    check_ctx(ctx);
    // the validation of fit_with_split (proj/src/embed.cpp:115-130)
    if (s < 0 || s > d)
      fail(ADG_EINVAL, "fit_with_split: s = " + std::to_string(s) + " outside [0, " +
                           std::to_string(d) + "]");
    if (k < 1)
      fail(ADG_EINVAL,
           "fit_with_split: k must be >= 1 (for a pure principal projection use the sweep "
           "module's pca method)");
    if (n_total < 2) fail(ADG_EINVAL, "fit_with_split: need at least 2 points");
    if (s + k > d)
      std::cerr << "fit_with_split: warning: output dimension " << (s + k)
                << " exceeds ambient dimension " << d << "\n";
    In g(gram, sizeof(double) * (size_t)(d * d), ctx->stream);
    Out b(basis_out, sizeof(double) * (size_t)(s * d), ctx->stream);
    Out sk(sketch_out, sizeof(double) * (size_t)(k * d), ctx->stream);
    if (s > 0) {
      const int64_t max_rank = std::min(n_total, d);
      if (s <= max_rank && backend == ADG_BACKEND_RANDOMIZED) {
        const int64_t over = std::min<int64_t>(10, max_rank - s);
        spectral_randomized_gram(ctx, g.as<double>(), d, s, over, 2, derive_seed(seed, "spectral"),
                                 b.as<double>(), nullptr);
      } else {
        spectral_exact_gram(ctx, g.as<double>(), d, s, b.as<double>());
      }
    }
    sample_jl_device(ctx, k, d, derive_seed(seed, "jl"), sk.as<double>());
    b.commit();
    sk.commit();
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// proj/src/embed.cpp:105-113
adg_status adg_fit(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                   int64_t target_dim, adg_backend backend, uint64_t seed, double* mean_out,
                   double* basis_out, double* sketch_out) {
  if (target_dim < 2 || target_dim > d) {
    set_last_error("fit: target_dim = " + std::to_string(target_dim) + " outside [2, " +
                   std::to_string(d) + "]");
    return ADG_EINVAL;
  }
  if (n < 2) {
    set_last_error("fit: need at least 2 points");
    return ADG_EINVAL;
  }
  return adg_fit_with_split(ctx, X, dtype, n, d, target_dim / 2, target_dim - target_dim / 2,
                            backend, seed, mean_out, basis_out, sketch_out);
}

// proj/src/embed.cpp:161-181
adg_status adg_transform_all(adg_ctx* ctx, const double* mean, const double* basis, int64_t s,
                             const double* sketch, int64_t k, int64_t d, const void* X,
                             adg_dtype dtype, int64_t n, void* Y_out, adg_dtype out_dtype) {
  return guard([&] {
    NvtxRange nvtx_("adg_transform_all");
    check_ctx(ctx);
    ADG_REQUIRE(s >= 0 && k >= 1 && d >= 1, "transform_all: invalid model dimensions");
    ADG_REQUIRE(n >= 0, "transform_all: negative row count");
    In mu(mean, sizeof(double) * (size_t)d, ctx->stream);
    In P(basis, sizeof(double) * (size_t)(s * d), ctx->stream);
    In S(sketch, sizeof(double) * (size_t)(k * d), ctx->stream);
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    Out y(Y_out, (size_t)(n * (s + k)) * dtype_size(out_dtype), ctx->stream);
    TransformPlan plan(ctx, mu.as<double>(), P.as<double>(), s, S.as<double>(), k, d,
                       dtype == ADG_F64);
    plan.run(x.dev, dtype, n, y.dev, out_dtype);
    y.commit();
    // device-resident output: stream-ordered, no host synchronisation needed
    if (y.staged.ptr) ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"

struct adg_transform_plan {
  adg_ctx* ctx;
  int64_t s, k, d;
  bool fp64;
  std::unique_ptr<adg::TransformPlan> plan;
};

extern "C" {

adg_status adg_transform_plan_create(adg_ctx* ctx, const double* mean, const double* basis,
                                     int64_t s, const double* sketch, int64_t k, int64_t d,
                                     adg_dtype input_dtype, adg_transform_plan** out) {
  return guard([&] {
    check_ctx(ctx);
    ADG_REQUIRE(out, "transform_plan_create: null output");
    ADG_REQUIRE(s >= 0 && k >= 1 && d >= 1, "transform_all: invalid model dimensions");
    In mu(mean, sizeof(double) * (size_t)d, ctx->stream);
    In P(basis, sizeof(double) * (size_t)(s * d), ctx->stream);
    In S(sketch, sizeof(double) * (size_t)(k * d), ctx->stream);
    auto p = std::make_unique<adg_transform_plan>();
    p->ctx = ctx;
    p->s = s;
    p->k = k;
    p->d = d;
    p->fp64 = input_dtype == ADG_F64;
    p->plan = std::make_unique<TransformPlan>(ctx, mu.as<double>(), P.as<double>(), s, S.as<double>(),
                                              k, d, p->fp64);
    // host-staged model constants are freed with `mu`, `P`, `S`: finish first
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = p.release();
  });
}

adg_status adg_transform_plan_run(adg_transform_plan* p, const void* X, adg_dtype dtype, int64_t n,
                                  void* Y_out, adg_dtype out_dtype) {
  return guard([&] {
    ADG_REQUIRE(p, "transform_plan_run: null plan");
    adg_ctx* ctx = p->ctx;
    ADG_CUDA(cudaSetDevice(ctx->device));
    ADG_REQUIRE(n >= 0, "transform_all: negative row count");
    if ((dtype == ADG_F64) != p->fp64)
      fail(ADG_EINVAL, "transform_plan_run: plan was built for " +
                           std::string(p->fp64 ? "fp64" : "fp32/bf16") + " input");
    In x(X, (size_t)(n * p->d) * dtype_size(dtype), ctx->stream);
    Out y(Y_out, (size_t)(n * (p->s + p->k)) * dtype_size(out_dtype), ctx->stream);
    p->plan->run(x.dev, dtype, n, y.dev, out_dtype);
    y.commit();
    if (y.staged.ptr) ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adg_status adg_transform_plan_destroy(adg_transform_plan* p) {
  return guard([&] {
    if (!p) return;
    cudaSetDevice(p->ctx->device);
    cudaStreamSynchronize(p->ctx->stream);
    delete p;
  });
}

}  // extern "C"

// Validation of evaluate()'s arguments (proj/src/distortion.cpp:116-122, :131-134).
static void check_evaluate_args(int64_t n, int64_t n_emb, const adg_pair_sampling* mode,
                                int hist_bins, double hist_max, const void* report,
                                const void* hist_out) {
  if (n != n_emb)
    fail(ADG_EINVAL, "evaluate: cloud sizes differ (" + std::to_string(n) + " vs " +
                         std::to_string(n_emb) + ")");
  if (hist_bins < 1 || !(hist_max > 0.0))
    fail(ADG_EINVAL, "evaluate: need hist_bins >= 1 and hist_max > 0");
  ADG_REQUIRE(report && hist_out, "evaluate: null report/hist");
  if (mode && !mode->all_pairs) {
    const uint64_t un = (uint64_t)std::max<int64_t>(n, 0);
    const uint64_t total_pairs = un * (un - (un ? 1 : 0)) / 2;
    if (mode->m < 1 || mode->m > total_pairs)
      fail(ADG_EINVAL, "evaluate: sample size " + std::to_string(mode->m) + " outside [1, " +
                           std::to_string(total_pairs) + "]");
  }
}

// proj/src/distortion.cpp:113-192 on device-resident clouds.
void adg::evaluate_device(adg_ctx* ctx, const void* xdev, adg_dtype orig_dtype, int64_t n,
                          int64_t d, const void* ydev, adg_dtype emb_dtype, int64_t r,
                          const adg_pair_sampling* mode, int hist_bins, double hist_max,
                          adg_engine engine, adg_report* report, uint64_t* hist_out) {
  const bool all_pairs = !mode || mode->all_pairs;
  const uint64_t un = (uint64_t)std::max<int64_t>(n, 0);
  const uint64_t total_pairs = un * (un - (un ? 1 : 0)) / 2;
  adg_report rep;
  std::memset(&rep, 0, sizeof(rep));
  std::vector<uint64_t> hist((size_t)hist_bins + 1, 0);
  if (!all_pairs) {
    std::vector<uint64_t> idx = sample_pair_indices(total_pairs, mode->m, mode->seed);
    DevBuf<uint64_t> idx_dev(idx.size(), ctx->stream);
    ADG_CUDA(cudaMemcpyAsync(idx_dev.ptr, idx.data(), idx.size() * sizeof(uint64_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    evaluate_exact(ctx, xdev, orig_dtype, n, d, ydev, emb_dtype, r, idx_dev.ptr,
                   (uint64_t)idx.size(), hist_bins, hist_max, &rep, hist.data());
    rep.sampled = 1;
    rep.sample_seed = mode->seed;
  } else {
    bool use_screen = engine == ADG_ENGINE_SCREEN || engine == ADG_ENGINE_SCREEN_EXACT_HIST ||
                      (engine == ADG_ENGINE_AUTO && n > 4096);
    if (n < 2 || d < 1 || r < 1) use_screen = false;
    if (use_screen) {
      adg_eval_plan* plan = cached_plan(ctx, xdev, orig_dtype, n, d, ydev, emb_dtype, r, hist_bins, hist_max);
      plan->edge_f = (float)screen_edge_band(engine == ADG_ENGINE_SCREEN_EXACT_HIST);
      try {
        plan_run(plan, 0, plan->ops->num_tiles);
        plan_finalize(plan, &rep, hist.data());
      } catch (...) {
        release_plan(ctx, plan);
        throw;
      }
      release_plan(ctx, plan);
    } else {
      evaluate_exact(ctx, xdev, orig_dtype, n, d, ydev, emb_dtype, r, nullptr, total_pairs,
                     hist_bins, hist_max, &rep, hist.data());
    }
  }
  rep.hist_bins = hist_bins;
  rep.hist_max = hist_max;
  *report = rep;
  std::memcpy(hist_out, hist.data(), hist.size() * sizeof(uint64_t));
}

double adg::max_distortion_device(adg_ctx* ctx, const void* xdev, adg_dtype xd, int64_t n,
                                 int64_t d, const void* ydev, adg_dtype yd, int64_t r,
                                 const adg_pair_sampling* mode, double* upper) {
  adg_report rep;
  std::vector<uint64_t> hist(2);
  const bool all_pairs = !mode || mode->all_pairs;
  if (all_pairs && n > 4096 && d >= 1 && r >= 1) {
    adg_eval_plan* plan = cached_plan(ctx, xdev, xd, n, d, ydev, yd, r, 1, 1.0);
    try {
      plan_run(plan, 0, plan->ops->num_tiles, /*max_only=*/true);
      if (upper) *upper = -1.0;
      plan_finalize(plan, &rep, hist.data(), upper);
    } catch (...) {
      release_plan(ctx, plan);
      throw;
    }
    release_plan(ctx, plan);
    return rep.max_distortion;
  }
  evaluate_device(ctx, xdev, xd, n, d, ydev, yd, r, mode, 1, 1.0, ADG_ENGINE_AUTO, &rep,
                  hist.data());
  if (upper) *upper = rep.max_distortion;
  return rep.max_distortion;
}

extern "C" {

// proj/src/distortion.cpp:113-192
adg_status adg_evaluate(adg_ctx* ctx, const void* orig, adg_dtype orig_dtype, int64_t n,
                        int64_t d, const void* emb, adg_dtype emb_dtype, int64_t n_emb,
                        int64_t r, const adg_pair_sampling* mode, int hist_bins,
                        double hist_max, uint64_t pairs_per_block, adg_engine engine,
                        adg_report* report, uint64_t* hist_out) {
  (void)pairs_per_block;  // results-neutral by contract (distortion.hpp:47-51)
  return guard([&] {
    NvtxRange nvtx_("adg_evaluate");
    check_ctx(ctx);
    check_evaluate_args(n, n_emb, mode, hist_bins, hist_max, report, hist_out);
    In x(orig, (size_t)(n * d) * dtype_size(orig_dtype), ctx->stream);
    In y(emb, (size_t)(n * r) * dtype_size(emb_dtype), ctx->stream);
    evaluate_device(ctx, x.dev, orig_dtype, n, d, y.dev, emb_dtype, r, mode, hist_bins, hist_max,
                    engine, report, hist_out);
  });
}

static bool is_pinned_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// run_distort --model with X in pinned host memory, all pairs, SCREEN engine:
// X crosses PCIe in row chunks on a copy stream while the compute stream
// embeds and preps each chunk and screens every tile whose rows have all
// arrived (tiles are phased by the rows they read).  The centring shift is
// computed first from the same <= kShiftRows evenly spaced rows the one-shot path
// uses (one strided copy), and tile partial sums sit in canonical slots, so
// the report is bit-identical to transform_all + evaluate.
// model of the pipelined flow for its phase grouping (adg_distort_model):
// host->device rate of pinned memory (B200 PCIe 5 x16 measures ~55 GB/s) and
// the screen's executed f16 rate
constexpr double kPipePcieBytesPerUs = 50e3;
constexpr double kPipeScreenTflops = 1500.0;

static void distort_pipelined(adg_ctx* ctx, const double* mu, const double* Pm, int64_t s,
                              const double* Sm, int64_t k, int64_t d, const void* X,
                              adg_dtype dtype, int64_t n, int hist_bins, double hist_max,
                              adg_report* report, uint64_t* hist_out, void* Y_out,
                              adg_dtype y_dtype, bool exact_hist) {
  const int64_t r = s + k;
  const size_t sx = dtype_size(dtype), sy = dtype_size(y_dtype);
  // ADG_PIPE_PROFILE=1: event timeline to stderr (profiling aid)
  const bool prof = std::getenv("ADG_PIPE_PROFILE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> tl;
  auto tmark = [&](const std::string& what, cudaStream_t st) {
    if (!prof) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tl.emplace_back(what, e);
  };
  const auto host_t0 = std::chrono::steady_clock::now();
  std::vector<std::pair<std::string, double>> htl;
  auto hmark = [&](const char* what) {
    if (prof)
      htl.emplace_back(what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count());
  };
  tmark("start", ctx->stream);
  DevBuf<uint8_t> xdev((size_t)(n * d) * sx, ctx->stream), ydev((size_t)(n * r) * sy, ctx->stream);
  // centring shift: column_means_sampled's rows, gathered by one strided copy
  const int64_t step = std::max<int64_t>(1, (n + kShiftRows - 1) / kShiftRows);
  const int64_t m = (n - 1) / step + 1;
  DevBuf<uint8_t> xs((size_t)(m * d) * sx, ctx->stream), ys((size_t)(m * r) * sy, ctx->stream);
  DevBuf<double> mx((size_t)d, ctx->stream), my((size_t)r, ctx->stream);
  // the chunk copies need only xdev's allocation: start them now, under the
  // centring-shift setup below
  if (!ctx->copy_stream) ADG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  // On every exit (an error included), before the buffers above are released
  // (stream-ordered on ctx->stream): drain the copy stream that writes into
  // them and the phase streams that read them, and destroy the events.
  struct PipeGuard {
    adg_ctx* ctx;
    std::vector<cudaEvent_t> events;
    ~PipeGuard() {
      cudaStreamSynchronize(ctx->copy_stream);
      for (cudaStream_t s : ctx->phase_streams)
        if (s) cudaStreamSynchronize(s);
      for (cudaEvent_t e : events) cudaEventDestroy(e);
    }
  } guard_{ctx, {}};
  cudaEvent_t ready;
  ADG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  guard_.events.push_back(ready);
  ADG_CUDA(cudaEventRecord(ready, ctx->stream));
  ADG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ready, 0));
  // the sampled rows first (copy engines serve H2D in issue order), then the chunks
  ADG_CUDA(cudaMemcpy2DAsync(xs.ptr, d * sx, X, step * d * sx, d * sx, m, cudaMemcpyHostToDevice,
                             ctx->copy_stream));
  cudaEvent_t sampled;
  ADG_CUDA(cudaEventCreateWithFlags(&sampled, cudaEventDisableTiming));
  guard_.events.push_back(sampled);
  ADG_CUDA(cudaEventRecord(sampled, ctx->copy_stream));
  // row chunks (multiples of the 256-row pair block) and the phased tile list
  const int64_t rows_pad = std::max((n + 255) / 256 * 256, (n + 159) / 160 * 160);  // as ScreenOperands
  const char* kc = std::getenv("ADG_PIPE_CHUNKS");  // profiling aid
  const int64_t K = std::max<int64_t>(1, std::min<int64_t>(kc ? std::atoll(kc) : 16, rows_pad / 2048));
  // chunk q ends at rows_pad (q/K)^p: p > 1 makes the first chunks smaller, so
  // the screen starts sooner (its work grows with the square of the rows in)
  const char* pe = std::getenv("ADG_PIPE_POWER");  // profiling aid
  const double pw = pe ? std::atof(pe) : 1.0;
  std::vector<int64_t> bounds;
  for (int64_t q = 1; q <= K; ++q) {
    const double f = std::pow((double)q / (double)K, pw);
    const int64_t b = std::min(rows_pad, ((int64_t)(f * (double)rows_pad) + 255) / 256 * 256);
    bounds.push_back(std::max<int64_t>(b, bounds.empty() ? 256 : bounds.back() + 256));
  }
  for (auto& b : bounds) b = std::min(b, rows_pad);
  bounds.back() = rows_pad;
  // the row chunks, queued at once behind the sampled rows: the copy engine
  // starts on them while the host builds the operands and plans below
  std::vector<cudaEvent_t> ev((size_t)K);
  int64_t prev = 0;
  for (int64_t q = 0; q < K; ++q) {
    const int64_t r1 = std::min(bounds[(size_t)q], n);
    ADG_CUDA(cudaEventCreateWithFlags(&ev[(size_t)q], cudaEventDisableTiming));
    guard_.events.push_back(ev[(size_t)q]);
    if (r1 > prev)
      ADG_CUDA(cudaMemcpyAsync(xdev.ptr + prev * d * sx, static_cast<const uint8_t*>(X) + prev * d * sx,
                               (size_t)((r1 - prev) * d) * sx, cudaMemcpyHostToDevice, ctx->copy_stream));
    ADG_CUDA(cudaEventRecord(ev[(size_t)q], ctx->copy_stream));
    tmark("h2d" + std::to_string(q), ctx->copy_stream);
    prev = std::max(prev, r1);
  }
  // planes, maps and the phased tile list (cached per context after the
  // first call).  Screen phases end at chunk ends, grouped by a model of the
  // flow: while the GPU waits on PCIe (early chunks: the work grows with the
  // square of the rows in) every chunk is a phase; once it is compute-bound a
  // phase takes every chunk that will have arrived when the GPU gets to it,
  // so fewer launch ramps and tails, and its chunks are embedded and prepared
  // in one launch pair (C3: 7.54 ms against 7.59 ms with one phase per chunk).
  // Any grouping gives the same report (phases update the partials
  // order-free).  ADG_PIPE_GROUP=0 (profiling aid): one phase per chunk.
  std::vector<int64_t> phase_end_chunk, phase_rows;
  {
    const char* pg = std::getenv("ADG_PIPE_GROUP");
    const bool group = !(pg && std::atoi(pg) == 0);
    const double pcie = kPipePcieBytesPerUs;  // conservative host->device rate
    const int64_t kpad = ((d + 15) / 16 + (r + 15) / 16) * 16;
    const double passes = dtype == ADG_BF16 ? 1.0 : 3.0;  // bf16: one-pass original side
    const double tile_us = 2.0 * 256 * 160 * (double)kpad * passes / (kPipeScreenTflops * 1e6);
    auto pairs_tiles = [&](int64_t rows) {  // tiles whose rows are all < rows (triangle)
      const double b = (double)rows / 256.0;
      return 0.5 * b * b * (256.0 / 160.0);
    };
    const double bytes_row = (double)(d * sx);
    double gpu_free = -1.0;
    int64_t q = 0;
    while (q < K) {
      const double arr_q = ((double)(m + std::min(bounds[(size_t)q], n))) * bytes_row / pcie;
      const double start = std::max(gpu_free, arr_q);
      int64_t e = q;
      if (group)
        while (e + 1 < K &&
               ((double)(m + std::min(bounds[(size_t)(e + 1)], n))) * bytes_row / pcie <= start)
          ++e;
      const int64_t rows0 = q ? bounds[(size_t)q - 1] : 0;
      gpu_free = start + (pairs_tiles(bounds[(size_t)e]) - pairs_tiles(rows0)) * tile_us;
      phase_end_chunk.push_back(e);
      phase_rows.push_back(bounds[(size_t)e]);
      q = e + 1;
    }
  }
  hmark("chunks enqueued");
  auto ops = std::make_unique<ScreenOperands>(ctx, n, d, r, &phase_rows);
  hmark("operands");
  ScreenOperands* op = ops.get();
  TransformPlan tp(ctx, mu, Pm, s, Sm, k, d, dtype == ADG_F64);  // under the copies
  hmark("transform plan");
  ADG_CUDA(cudaStreamWaitEvent(ctx->stream, sampled, 0));
  tp.run(xs.ptr, dtype, m, ys.ptr, y_dtype);
  screen_shift(ctx, xs.ptr, dtype, m, d, mx.ptr);  // the same rows as ScreenOperands samples
  column_means_sampled(ctx, ys.ptr, y_dtype, m, r, kShiftRows, my.ptr);
  tmark("shift", ctx->stream);
  std::unique_ptr<adg_eval_plan> plan(plan_create(ctx, xdev.ptr, dtype, n, d, ydev.ptr, y_dtype, r,
                                                  hist_bins, hist_max, std::move(ops)));
  hmark("plan");
  plan->edge_f = (float)screen_edge_band(exact_hist);
  // the phases run on other streams: the edge list must exist before the
  // events they wait on (stream-ordered allocation on the context stream)
  if (plan->edge_f > 0.f) plan->edge_pairs.alloc((size_t)plan->edge_cap, ctx->stream);
  // Phase q's screen runs on phase stream q % 2 as soon as its rows are
  // prepared, so it overlaps the previous phase's drain (the screen launches
  // are persistent grids: their tails leave SMs idle) and the next chunk's
  // embedding and prep.  Phases read disjoint tiles and update the partials
  // order-free (integer / max atomics, one writer per tile-sum slot); the edge
  // list is binned once after all of them.
  for (cudaStream_t& s : ctx->phase_streams)
    if (!s) ADG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const char* pse = std::getenv("ADG_PIPE_STREAMS");  // profiling aid
  const size_t nps = (size_t)std::max(1, std::min(4, pse ? std::atoi(pse) : 2));
  std::vector<cudaEvent_t> prepped((size_t)K);
  for (auto& e : prepped) {
    ADG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    guard_.events.push_back(e);
  }
  // each phase embeds and prepares the rows of its chunks in one launch pair
  // once its last chunk is in, then screens its tiles
  int64_t lo = 0;
  for (size_t ph = 0; ph < phase_end_chunk.size(); ++ph) {
    const int64_t q = phase_end_chunk[ph];
    const int64_t hi_pad = bounds[(size_t)q], r1 = std::min(hi_pad, n);
    ADG_CUDA(cudaStreamWaitEvent(ctx->stream, ev[(size_t)q], 0));
    if (r1 > lo)
      tp.run(xdev.ptr + lo * d * sx, dtype, r1 - lo, ydev.ptr + lo * r * sy, y_dtype);
    op->prep_rows(xdev.ptr, dtype, ydev.ptr, y_dtype, mx.ptr, my.ptr, lo, hi_pad);
    tmark("prep" + std::to_string(ph), ctx->stream);
    lo = hi_pad;
    ADG_CUDA(cudaEventRecord(prepped[ph], ctx->stream));
    cudaStream_t ps = ctx->phase_streams[ph % nps];
    ADG_CUDA(cudaStreamWaitEvent(ps, prepped[ph], 0));
    plan_screen(plan.get(), ph == 0 ? 0 : op->phase_tile_end[ph - 1], op->phase_tile_end[ph], false, ps);
    tmark("screen" + std::to_string(ph), ps);
  }
  for (cudaStream_t ps : ctx->phase_streams) {  // join
    cudaEvent_t done;
    ADG_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    guard_.events.push_back(done);
    ADG_CUDA(cudaEventRecord(done, ps));
    ADG_CUDA(cudaStreamWaitEvent(ctx->stream, done, 0));
  }
  hmark("phases enqueued");
  plan_edge_bin(plan.get());
  if (Y_out) ADG_CUDA(cudaMemcpyAsync(Y_out, ydev.ptr, ydev.count, cudaMemcpyDefault, ctx->stream));
  adg_report rep;
  std::vector<uint64_t> hist((size_t)hist_bins + 1, 0);
  plan_finalize(plan.get(), &rep, hist.data());
  rep.hist_bins = hist_bins;
  rep.hist_max = hist_max;
  *report = rep;
  std::memcpy(hist_out, hist.data(), hist.size() * sizeof(uint64_t));
  hmark("finalized");
  ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (prof) {
    hmark("synced");
    for (auto& h : htl) std::fprintf(stderr, "[pipe] host %-18s %8.3f ms\n", h.first.c_str(), h.second);
    tmark("end", ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    const double host_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    for (auto& pe : tl) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tl.front().second, pe.second);
      std::fprintf(stderr, "[pipe] %-9s %8.3f ms\n", pe.first.c_str(), ms);
    }
    for (auto& pe : tl) cudaEventDestroy(pe.second);
    std::fprintf(stderr, "[pipe] host wall %.3f ms, tiles per phase:", host_ms);
    for (size_t q = 0; q < op->phase_tile_end.size(); ++q)
      std::fprintf(stderr, " %lld", (long long)(op->phase_tile_end[q] - (q ? op->phase_tile_end[q - 1] : 0)));
    std::fprintf(stderr, "\n");
  }
}

// proj/tools/adagio_main.cpp:192-224 (run_distort with --model): transform_all
// of the original cloud, then evaluate(original, embedded).  The original is
// staged to the device once and the embedding never leaves HBM unless Y_out
// asks for it -- the reference's value-semantics flow without the second copy.
adg_status adg_distort_model(adg_ctx* ctx, const double* mean, const double* basis, int64_t s,
                             const double* sketch, int64_t k, int64_t d, const void* X,
                             adg_dtype dtype, int64_t n, const adg_pair_sampling* mode,
                             int hist_bins, double hist_max, adg_engine engine,
                             adg_report* report, uint64_t* hist_out, void* Y_out,
                             adg_dtype y_dtype) {
  return guard([&] {
    NvtxRange nvtx_("adg_distort_model");
    struct EntryClock {  // ADG_PIPE_PROFILE: whole-call host time (profiling aid)
      std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
      ~EntryClock() {
        if (std::getenv("ADG_PIPE_PROFILE"))
          std::fprintf(stderr, "[pipe] call wall %.3f ms\n",
                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      }
    } entry_clock_;
    check_ctx(ctx);
    ADG_REQUIRE(s >= 0 && k >= 1 && d >= 1, "transform_all: invalid model dimensions");
    ADG_REQUIRE(n >= 0, "transform_all: negative row count");
    ADG_REQUIRE(y_dtype == ADG_F32 || y_dtype == ADG_F64, "distort: embedding dtype must be f32/f64");
    const int64_t r = s + k;
    check_evaluate_args(n, n, mode, hist_bins, hist_max, report, hist_out);
    In mu(mean, sizeof(double) * (size_t)d, ctx->stream);
    In P(basis, sizeof(double) * (size_t)(s * d), ctx->stream);
    In S(sketch, sizeof(double) * (size_t)(k * d), ctx->stream);
    const bool all_pairs = !mode || mode->all_pairs;
    const bool screen = engine == ADG_ENGINE_SCREEN || engine == ADG_ENGINE_SCREEN_EXACT_HIST ||
                        (engine == ADG_ENGINE_AUTO && n > 4096);
    if (all_pairs && screen && n >= 4096 && is_pinned_host(X)) {
      if (std::getenv("ADG_PIPE_PROFILE"))
        std::fprintf(stderr, "[pipe] call setup %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - entry_clock_.t0).count());
      distort_pipelined(ctx, mu.as<double>(), P.as<double>(), s, S.as<double>(), k, d, X, dtype, n,
                        hist_bins, hist_max, report, hist_out, Y_out, y_dtype,
                        engine == ADG_ENGINE_SCREEN_EXACT_HIST);
      if (std::getenv("ADG_PIPE_PROFILE"))
        std::fprintf(stderr, "[pipe] call pipelined done %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - entry_clock_.t0).count());
      return;
    }
    In x(X, (size_t)(n * d) * dtype_size(dtype), ctx->stream);
    DevBuf<uint8_t> ydev((size_t)(n * r) * dtype_size(y_dtype), ctx->stream);
    {
      TransformPlan plan(ctx, mu.as<double>(), P.as<double>(), s, S.as<double>(), k, d,
                         dtype == ADG_F64);
      plan.run(x.dev, dtype, n, ydev.ptr, y_dtype);
    }
    if (Y_out)
      ADG_CUDA(cudaMemcpyAsync(Y_out, ydev.ptr, ydev.count, cudaMemcpyDefault, ctx->stream));
    evaluate_device(ctx, x.dev, dtype, n, d, ydev.ptr, y_dtype, r, mode, hist_bins, hist_max,
                    engine, report, hist_out);
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// proj/src/distortion.cpp:194-196
adg_status adg_max_distortion(adg_ctx* ctx, const void* orig, adg_dtype orig_dtype, int64_t n,
                              int64_t d, const void* emb, adg_dtype emb_dtype, int64_t r,
                              double* out) {
  return guard([&] {
    check_ctx(ctx);
    check_evaluate_args(n, n, nullptr, 1, 1.0, out, out);
    In x(orig, (size_t)(n * d) * dtype_size(orig_dtype), ctx->stream);
    In y(emb, (size_t)(n * r) * dtype_size(emb_dtype), ctx->stream);
    *out = max_distortion_device(ctx, x.dev, orig_dtype, n, d, y.dev, emb_dtype, r, nullptr);
  });
}

// proj/src/distortion.cpp:107-111
adg_status adg_pair_distortion(adg_ctx* ctx, const double* x, const double* y, int64_t d,
                               const double* fx, const double* fy, int64_t r, double* out) {
  return guard([&] {
    check_ctx(ctx);
    ADG_REQUIRE(d >= 1 && r >= 1 && out, "pair_distortion: bad arguments");
    std::vector<double> X((size_t)(2 * d)), Y((size_t)(2 * r));
    std::memcpy(X.data(), x, sizeof(double) * d);
    std::memcpy(X.data() + d, y, sizeof(double) * d);
    std::memcpy(Y.data(), fx, sizeof(double) * r);
    std::memcpy(Y.data() + r, fy, sizeof(double) * r);
    In xd(X.data(), X.size() * sizeof(double), ctx->stream);
    In yd(Y.data(), Y.size() * sizeof(double), ctx->stream);
    uint32_t pair[2] = {0, 1};
    In pd(pair, sizeof(pair), ctx->stream);
    DevBuf<double> v(1, ctx->stream);
    run_pair_list(ctx, xd.dev, ADG_F64, d, yd.dev, ADG_F64, r, pd.as<uint32_t>(), 1, v.ptr);
    double h = 0.0;
    ADG_CUDA(cudaMemcpyAsync(&h, v.ptr, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ADG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h < 0.0) fail(ADG_EINVAL, "pair_distortion: coincident points");
    *out = h;
  });
}

static size_t emit(char* buf, size_t cap, const std::string& s) {
  if (buf && cap) {
    const size_t k = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return s.size();
}

static std::string fmt17(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

// proj/src/distortion.cpp:198-215 (keys of proj/docs/schemas/distort.schema.json)
size_t adg_report_to_json(const adg_report* r, const uint64_t* hist, char* buf, size_t cap) {
  std::string s = "{\"max_distortion\":" + fmt17(r->max_distortion) +
                  ",\"mean_distortion\":" + fmt17(r->mean_distortion) +
                  ",\"hist_bins\":" + std::to_string(r->hist_bins) + ",\"hist_max\":" +
                  fmt17(r->hist_max) + ",\"histogram\":[";
  for (int b = 0; b <= r->hist_bins; ++b) s += (b ? "," : "") + std::to_string(hist[b]);
  s += "],\"n_pairs_evaluated\":" + std::to_string(r->n_pairs_evaluated) +
       ",\"n_zero_distance_pairs\":" + std::to_string(r->n_zero_distance_pairs) +
       ",\"sampled\":" + (r->sampled ? "true" : "false") + ",\"sample_seed\":" +
       (r->sampled ? std::to_string(r->sample_seed) : std::string("null"));
  if (r->argmax_i != UINT64_MAX)
    s += ",\"argmax_i\":" + std::to_string(r->argmax_i) + ",\"argmax_j\":" +
         std::to_string(r->argmax_j);
  s += "}";
  return emit(buf, cap, s);
}

// proj/src/distortion.cpp:217-230
size_t adg_histogram_csv(const adg_report* r, const uint64_t* hist, char* buf, size_t cap) {
  std::string out = "bin_left,bin_right,count\n";
  char line[96];
  const double width = r->hist_max / r->hist_bins;
  for (int b = 0; b < r->hist_bins; ++b) {
    std::snprintf(line, sizeof(line), "%.17g,%.17g,%llu\n", b * width, (b + 1) * width,
                  (unsigned long long)hist[b]);
    out += line;
  }
  std::snprintf(line, sizeof(line), "%.17g,inf,%llu\n", r->hist_max,
                (unsigned long long)hist[r->hist_bins]);
  out += line;
  return emit(buf, cap, out);
}

// --------------------------------------------------------- sharded plans
adg_status adg_eval_plan_create(adg_ctx* ctx, const void* orig, adg_dtype orig_dtype, int64_t n,
                                int64_t d, const void* emb, adg_dtype emb_dtype, int64_t r,
                                int hist_bins, double hist_max, adg_eval_plan** out) {
  return guard([&] {
    check_ctx(ctx);
    if (hist_bins < 1 || !(hist_max > 0.0))
      fail(ADG_EINVAL, "evaluate: need hist_bins >= 1 and hist_max > 0");
    ADG_REQUIRE(n >= 2 && d >= 1 && r >= 1 && out, "evaluate: plan needs n >= 2, d, r >= 1");
    *out = plan_create(ctx, orig, orig_dtype, n, d, emb, emb_dtype, r, hist_bins, hist_max);
    // device inputs: the operand prep stays queued on the stream (the sharded
    // evaluator enqueues run / exchange / finalize behind it); host inputs
    // were staged asynchronously from caller memory, so wait for those copies
    if ((*out)->orig->staged.ptr || (*out)->emb->staged.ptr) ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

adg_status adg_eval_plan_partials(adg_eval_plan* p, adg_eval_partials* out) {
  return guard([&] {
    ADG_REQUIRE(p && out, "null plan");
    out->hist = reinterpret_cast<uint64_t*>(p->hist());
    out->tile_sums = p->tile_sums.ptr;
    out->row_max = p->row_max_ptr();
    out->row_bound = p->row_bound_ptr();
    out->near_pairs = p->near_pairs.ptr;
    out->near_count = reinterpret_cast<uint64_t*>(p->near_count());
    out->num_tiles = p->ops->num_tiles;
    out->near_capacity = p->near_cap;
    out->n = p->n;
    out->hist_bins = p->bins;
    out->tile_slots = screen_tile_slots();
  });
}

adg_status adg_eval_plan_refresh(adg_eval_plan* p) {
  return guard([&] {
    ADG_REQUIRE(p, "null plan");
    check_ctx(p->ctx);
    ADG_REQUIRE(p->created_on == p->ctx->stream, "eval_plan_refresh: the context's stream changed");
    if (p->orig->staged.ptr || p->emb->staged.ptr)
      fail(ADG_EINVAL, "eval_plan_refresh: the plan was built from host buffers (staged copies)");
    plan_refresh(p);
  });
}

adg_status adg_eval_plan_reset(adg_eval_plan* p) {
  return guard([&] {
    ADG_REQUIRE(p, "null plan");
    check_ctx(p->ctx);
    plan_reset(p);
  });
}

adg_status adg_eval_plan_run(adg_eval_plan* p, int64_t tile_begin, int64_t tile_end) {
  return guard([&] {
    NvtxRange nvtx_("adg_eval_plan_run");
    ADG_REQUIRE(p, "null plan");
    check_ctx(p->ctx);
    ADG_REQUIRE(0 <= tile_begin && tile_begin <= tile_end && tile_end <= p->ops->num_tiles,
                "eval_plan_run: tile range outside [0, num_tiles]");
    plan_run(p, tile_begin, tile_end);
  });
}

adg_status adg_eval_plan_finalize(adg_eval_plan* p, adg_report* report, uint64_t* hist_out) {
  return guard([&] {
    NvtxRange nvtx_("adg_eval_plan_finalize");
    ADG_REQUIRE(p && report, "null plan/report");
    check_ctx(p->ctx);
    plan_finalize(p, report, hist_out);
  });
}

// Near-coincident list exchange: each rank packs [count, 0, pairs...]
// (block_pairs pairs) for one all-gather; the merge concatenates the gathered
// blocks in rank order into the plan's list.  A rank over its block, or a
// total over the plan's capacity, marks the list overflowed (count =
// capacity + 1: the finalize then redoes the histogram in tile chunks).
__global__ void near_pack_kernel(const uint32_t* __restrict__ pairs, const unsigned long long* __restrict__ count,
                                 int64_t block_pairs, int32_t* __restrict__ block) {
  const unsigned long long c = *count;
  const int64_t m = (int64_t)(c < (unsigned long long)block_pairs ? c : (unsigned long long)block_pairs);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < 2 * block_pairs + 2;
       t += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = 0;
    if (t == 0)
      v = (int32_t)(c > (unsigned long long)block_pairs ? block_pairs + 1 : c);
    else if (t >= 2 && (t - 2) < 2 * m)
      v = (int32_t)pairs[t - 2];
    block[t] = v;
  }
}

__global__ void near_merge_kernel(const int32_t* __restrict__ blocks, int world, int64_t block_pairs,
                                  int64_t cap, int regather, uint32_t* __restrict__ pairs,
                                  unsigned long long* __restrict__ count) {
  // one CTA per source rank; offsets from the counts before it (world is small)
  const int src = blockIdx.x;
  int64_t off = 0, total = 0;
  bool over_block = false;
  for (int w = 0; w < world; ++w) {
    const int64_t c = blocks[(int64_t)w * (2 * block_pairs + 2)];
    if (c > block_pairs) over_block = true;
    if (w < src) off += c;
    total += c;
  }
  const bool over = over_block || total > cap;
  if (!over) {
    const int64_t c = blocks[(int64_t)src * (2 * block_pairs + 2)];
    const int32_t* b = blocks + (int64_t)src * (2 * block_pairs + 2) + 2;
    for (int64_t t = threadIdx.x; t < 2 * c; t += blockDim.x) pairs[2 * off + t] = (uint32_t)b[t];
  }
  if (src == 0 && threadIdx.x == 0)
    *count = !over ? (unsigned long long)total
                   : (over_block && regather) ? kNearRegather : (unsigned long long)(cap + 1);
}

__global__ void init_rowbest_kernel(RowBest* __restrict__ rb, int64_t count) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x)
    rb[t] = RowBest{-1.0, -1, -1};
}
static void init_rowbest(adg_ctx* ctx, RowBest* rb, int64_t count) {
  init_rowbest_kernel<<<blocks_for(count, 256, 64), 256, 0, ctx->stream>>>(rb, count);
  after_launch(ctx);
}

// All-gather every rank's near-coincident list (own count in p->own_near)
// in blocks of g pairs and merge them in rank order into the plan's list.
static void near_gather(adg_eval_plan* p, const adg_collectives* c, int64_t g, bool regather) {
  adg_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  DevBuf<int32_t> block((size_t)(2 * g + 2), st), blocks((size_t)(c->world * (2 * g + 2)), st);
  near_pack_kernel<<<blocks_for(2 * g + 2, 256, 64), 256, 0, st>>>(p->near_pairs.ptr, p->own_near.ptr, g,
                                                                  block.ptr);
  after_launch(ctx);
  if (c->all_gather(c->user, block.ptr, blocks.ptr, (int64_t)sizeof(int32_t) * (2 * g + 2), st) != 0)
    fail(ADG_ENCCL, "eval_plan_exchange: all_gather(near pairs) failed");
  near_merge_kernel<<<(unsigned)c->world, 256, 0, st>>>(blocks.ptr, c->world, g, p->near_cap, regather ? 1 : 0,
                                                        p->near_pairs.ptr, p->near_count());
  after_launch(ctx);
}

// Second, sized gather (finalize, after kNearRegather): the largest count
// over the ranks sizes the blocks; above the plan's capacity -> overflow.
static unsigned long long near_regather(adg_eval_plan* p) {
  const adg_collectives* c = p->last_comm;
  if (!c) fail(ADG_EINVAL, "eval_plan_finalize: the exchange's collectives are needed again (near-coincident "
                           "lists larger than the first gather) but none was recorded");
  adg_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  DevBuf<unsigned long long> mx(1, st);
  ADG_CUDA(cudaMemcpyAsync(mx.ptr, p->own_near.ptr, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
  if (c->all_reduce(c->user, mx.ptr, 1, ADG_MAX_U64, st) != 0)
    fail(ADG_ENCCL, "eval_plan_finalize: all_reduce(near count) failed");
  unsigned long long most = 0;
  ADG_CUDA(cudaMemcpyAsync(&most, mx.ptr, sizeof(most), cudaMemcpyDeviceToHost, st));
  ADG_CUDA(cudaStreamSynchronize(st));
  if ((int64_t)most > p->near_cap) return most;  // a rank overflowed: chunked redo
  near_gather(p, c, (int64_t)most, false);
  unsigned long long merged = 0;
  ADG_CUDA(cudaMemcpyAsync(&merged, p->near_count(), sizeof(merged), cudaMemcpyDeviceToHost, st));
  ADG_CUDA(cudaStreamSynchronize(st));
  return merged;
}

// the one exchange of the sharded evaluator (also behind
// adg_evaluate_multi and the Python ShardedEvaluator).
static void plan_exchange(adg_eval_plan* p, const adg_collectives* c) {
  if (c->world <= 1) return;
  adg_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  auto call = [&](int rc, const char* what) {
    if (rc != 0)
      fail(ADG_ENCCL, std::string("eval_plan_exchange: ") + what + " failed (" + std::to_string(rc) + ")");
  };
  // [edge pairs binned | histogram] are contiguous in the stage block
  static_assert(adg_eval_plan::kHead == 6, "stage layout");
  call(c->all_reduce(c->user, p->edge_binned(), p->bins + 2, ADG_SUM_U64, st), "all_reduce(histogram)");
  call(c->all_reduce(c->user, p->tile_sums.ptr, screen_tile_slots() * p->ops->num_tiles, ADG_SUM_F64, st),
       "all_reduce(tile sums)");
  call(c->all_reduce(c->user, p->rows2.ptr, 2 * p->n, ADG_MAX_F32, st), "all_reduce(row maxima)");
  // the row holding the screened maximum (identical on every rank) and its
  // exact refine, its j chunks split over the ranks and all-gathered: the
  // finalize's lower bound L then needs no replicated row refine
  {
    argmax_f32(ctx, p->row_max_ptr(), p->n, p->best_row());
    const int64_t cpr = p->refine_chunks, W = c->world;
    const int64_t B = (cpr + W - 1) / W;  // chunks per rank
    const int64_t c0 = std::min(cpr, B * c->rank), c1 = std::min(cpr, c0 + B);
    DevBuf<RowBest> mine((size_t)B, st), all((size_t)(W * B), st);
    init_rowbest(ctx, mine.ptr, B);  // chunks past cpr stay "no pair"
    run_row_refine_chunks(ctx, p->orig->dev, p->xd, p->n, p->d, p->emb->dev, p->yd, p->r,
                          p->best_row(), c0, c1, mine.ptr);
    call(c->all_gather(c->user, mine.ptr, all.ptr, (int64_t)sizeof(RowBest) * B, st),
         "all_gather(row refine)");
    ADG_CUDA(cudaMemcpyAsync(p->best_row_refine(), all.ptr, sizeof(RowBest) * (size_t)cpr,
                             cudaMemcpyDeviceToDevice, st));
    p->best_refined = true;
  }
  // near-coincident lists: a fixed-size gather, stream-ordered (no host
  // round trip); a rank whose list does not fit marks it for the finalize,
  // which gathers again with the size the largest list needs
  if (!p->own_near.ptr) p->own_near.alloc(1, st);
  ADG_CUDA(cudaMemcpyAsync(p->own_near.ptr, p->near_count(), sizeof(unsigned long long),
                           cudaMemcpyDeviceToDevice, st));
  near_gather(p, c, std::min<int64_t>(p->near_cap, kNearBlock), true);
  p->last_comm = c;
}

static void shard_range(int64_t num_tiles, int world, int rank, int64_t* b, int64_t* e) {
  *b = num_tiles * rank / world;
  *e = num_tiles * (rank + 1) / world;
}

adg_status adg_eval_plan_set_engine(adg_eval_plan* p, adg_engine engine) {
  return guard([&] {
    ADG_REQUIRE(p, "null plan");
    ADG_REQUIRE(engine == ADG_ENGINE_AUTO || engine == ADG_ENGINE_SCREEN ||
                    engine == ADG_ENGINE_SCREEN_EXACT_HIST,
                "eval_plan_set_engine: a plan runs the SCREEN engine");
    p->edge_f = (float)screen_edge_band(engine == ADG_ENGINE_SCREEN_EXACT_HIST);
  });
}

adg_status adg_eval_plan_shard(adg_eval_plan* p, int32_t world, int32_t rank, int64_t* tile_begin,
                               int64_t* tile_end) {
  return guard([&] {
    ADG_REQUIRE(p && tile_begin && tile_end && world >= 1 && rank >= 0 && rank < world,
                "eval_plan_shard: bad arguments");
    shard_range(p->ops->num_tiles, world, rank, tile_begin, tile_end);
  });
}

adg_status adg_evaluate_multi(int32_t ndev, const int32_t* devices, const void* orig,
                              adg_dtype orig_dtype, int64_t n, int64_t d, const void* emb,
                              adg_dtype emb_dtype, int64_t n_emb, int64_t r,
                              const adg_pair_sampling* mode, int hist_bins, double hist_max,
                              adg_engine engine, adg_report* report, uint64_t* hist_out) {
  return guard([&] {
    NvtxRange nvtx_("adg_evaluate_multi");
    ADG_REQUIRE(ndev >= 1 && devices, "evaluate_multi: need ndev >= 1 devices");
    check_evaluate_args(n, n_emb, mode, hist_bins, hist_max, report, hist_out);
    const bool all_pairs = !mode || mode->all_pairs;
    const bool screen = all_pairs && n >= 2 && d >= 1 && r >= 1 &&
                        (engine == ADG_ENGINE_SCREEN || engine == ADG_ENGINE_SCREEN_EXACT_HIST ||
                         (engine == ADG_ENGINE_AUTO && n > 4096));
    struct CtxOwner {
      adg_ctx* c = nullptr;
      ~CtxOwner() { if (c) adg_ctx_destroy(c); }
    };
    if (ndev == 1 || !screen) {
      CtxOwner o;
      const adg_status s0 = adg_ctx_create(devices[0], &o.c);
      if (s0 != ADG_OK) fail(s0, g_last_error);
      In x(orig, (size_t)(n * d) * dtype_size(orig_dtype), o.c->stream);
      In y(emb, (size_t)(n * r) * dtype_size(emb_dtype), o.c->stream);
      evaluate_device(o.c, x.dev, orig_dtype, n, d, y.dev, emb_dtype, r, mode, hist_bins, hist_max,
                      engine, report, hist_out);
      return;
    }
    std::vector<adg_collectives> comms((size_t)ndev);
    {
      const adg_status s0 = adg_comm_nccl_create_all(ndev, devices, comms.data());
      if (s0 != ADG_OK) fail(s0, g_last_error);
    }
    std::vector<adg_status> status((size_t)ndev, ADG_OK);
    std::vector<std::string> errs((size_t)ndev);
    std::vector<adg_report> reps((size_t)ndev);
    std::vector<std::vector<uint64_t>> hists((size_t)ndev, std::vector<uint64_t>((size_t)hist_bins + 1));
    std::vector<std::thread> workers;
    for (int rank = 0; rank < ndev; ++rank)
      workers.emplace_back([&, rank] {
        status[(size_t)rank] = guard([&] {
          CtxOwner o;
          const adg_status s0 = adg_ctx_create(devices[rank], &o.c);
          if (s0 != ADG_OK) fail(s0, g_last_error);
          std::unique_ptr<adg_eval_plan> plan(
              plan_create(o.c, orig, orig_dtype, n, d, emb, emb_dtype, r, hist_bins, hist_max));
          plan->edge_f = (float)screen_edge_band(engine == ADG_ENGINE_SCREEN_EXACT_HIST);
          int64_t t0 = 0, t1 = 0;
          shard_range(plan->ops->num_tiles, ndev, rank, &t0, &t1);
          plan_run(plan.get(), t0, t1);
          plan_exchange(plan.get(), &comms[(size_t)rank]);
          plan_finalize(plan.get(), &reps[(size_t)rank], hists[(size_t)rank].data());
          reps[(size_t)rank].hist_bins = hist_bins;
          reps[(size_t)rank].hist_max = hist_max;
          ADG_CUDA(cudaStreamSynchronize(o.c->stream));
        });
        if (status[(size_t)rank] != ADG_OK) errs[(size_t)rank] = g_last_error;
      });
    for (auto& w : workers) w.join();
    for (auto& c : comms) adg_comm_nccl_destroy(&c);
    for (int rank = 0; rank < ndev; ++rank)
      if (status[(size_t)rank] != ADG_OK)
        fail(status[(size_t)rank], "evaluate_multi: rank " + std::to_string(rank) + ": " + errs[(size_t)rank]);
    *report = reps[0];
    std::memcpy(hist_out, hists[0].data(), hists[0].size() * sizeof(uint64_t));
  });
}

adg_status adg_eval_plan_exchange(adg_eval_plan* p, const adg_collectives* comm) {
  return guard([&] {
    NvtxRange nvtx_("adg_eval_plan_exchange");
    ADG_REQUIRE(p && comm && comm->all_reduce && comm->all_gather && comm->world >= 1,
                "eval_plan_exchange: bad arguments");
    check_ctx(p->ctx);
    plan_exchange(p, comm);
  });
}

adg_status adg_eval_plan_destroy(adg_eval_plan* p) {
  return guard([&] {
    if (!p) return;
    cudaSetDevice(p->ctx->device);
    cudaStreamSynchronize(p->ctx->stream);
    delete p;
  });
}

double adg_last_screen_kernel_ms(adg_ctx* ctx) {
  if (!ctx) return -1.0;
  if (ctx->last_screen_ms == -2.0) {
    float ms = 0.f;
    if (cudaEventSynchronize(ctx->ev_b) == cudaSuccess &&
        cudaEventElapsedTime(&ms, ctx->ev_a, ctx->ev_b) == cudaSuccess)
      ctx->last_screen_ms = ms;
    else
      ctx->last_screen_ms = -1.0;
  }
  return ctx->last_screen_ms;
}

uint64_t adg_kernel_launch_count(adg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int adg_last_knn_engine(adg_ctx* ctx) { return ctx ? ctx->last_knn_engine : 0; }

int adg_last_screen_orig_passes(adg_ctx* ctx) { return ctx ? ctx->last_orig_passes : 0; }

}  // extern "C"
