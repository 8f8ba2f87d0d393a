/*
 * adagio_oracle.c -- CPU restatement of the ADAgIO reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see adagio_oracle.h).  Plain C11 + pthreads,
 * fp64 throughout like the reference ("no 32-bit mode").
 * Compiled like the reference: -O3, no -march (proj/CMakeLists.txt:8-10,
 * proj/src/CMakeLists.txt:15).
 */
#include "adagio_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------ rng.hpp */

/* proj/include/adagio/rng.hpp:11-16 (splitmix64 finalizer). */
uint64_t or_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* proj/include/adagio/rng.hpp:19-26 */
uint64_t or_fnv1a64(const char* bytes, int64_t len) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < len; ++i) {
    h ^= (unsigned char)bytes[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* proj/include/adagio/rng.hpp:30-32 */
uint64_t or_derive_seed(uint64_t seed, const char* purpose) {
  return or_mix64(or_mix64(seed) ^ or_fnv1a64(purpose, (int64_t)strlen(purpose)));
}

/* proj/include/adagio/rng.hpp:37-39 */
uint64_t or_hash_position(uint64_t seed, uint64_t i, uint64_t j) {
  return or_mix64(or_mix64(or_mix64(seed) ^ i) ^ j);
}

/* proj/include/adagio/rng.hpp:42-44 */
double or_rademacher_sign(uint64_t seed, uint64_t i, uint64_t j) {
  return (or_hash_position(seed, i, j) >> 63) ? -1.0 : 1.0;
}

/* SeededRng, proj/include/adagio/rng.hpp:49-91 */
typedef struct {
  uint64_t state;
  double cached;
  int has_cached;
} seeded_rng;

static void rng_init(seeded_rng* r, uint64_t seed) {
  r->state = seed;
  r->cached = 0.0;
  r->has_cached = 0;
}

/* rng.hpp:53-58 */
static uint64_t rng_next_u64(seeded_rng* r) {
  uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:61-66 */
static uint64_t rng_below(seeded_rng* r, uint64_t bound) {
  const uint64_t limit = bound * ((~(uint64_t)0) / bound);
  uint64_t v = rng_next_u64(r);
  while (v >= limit) v = rng_next_u64(r);
  return v % bound;
}

/* rng.hpp:69 */
static double rng_unit(seeded_rng* r) { return (double)(rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:72-85 (Box-Muller, caches the sine deviate) */
static double rng_normal(seeded_rng* r) {
  if (r->has_cached) {
    r->has_cached = 0;
    return r->cached;
  }
  double u1 = rng_unit(r);
  while (u1 <= 0.0) u1 = rng_unit(r);
  const double u2 = rng_unit(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 6.283185307179586476925286766559 * u2;
  r->cached = radius * sin(angle);
  r->has_cached = 1;
  return radius * cos(angle);
}

void or_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
  seeded_rng r;
  rng_init(&r, seed);
  for (int64_t t = 0; t < count; ++t) out[t] = rng_next_u64(&r);
}

void or_rng_below(uint64_t seed, uint64_t bound, int64_t count, uint64_t* out) {
  seeded_rng r;
  rng_init(&r, seed);
  for (int64_t t = 0; t < count; ++t) out[t] = rng_below(&r, bound);
}

void or_rng_normal(uint64_t seed, int64_t count, double* out) {
  seeded_rng r;
  rng_init(&r, seed);
  for (int64_t t = 0; t < count; ++t) out[t] = rng_normal(&r);
}

/* ------------------------------------------------------ parallel_chunks */

/* proj/src/parallel.cpp:30-61: atomic-counter chunk claiming.  The callers
 * below write one result slot per chunk, so results never depend on the
 * worker count (proj/include/adagio/parallel.hpp:8-11). */
typedef void (*chunk_fn)(void* ctx, uint64_t chunk);
typedef struct {
  atomic_uint_fast64_t next;
  uint64_t count;
  chunk_fn fn;
  void* ctx;
} chunk_pool;

static void* chunk_worker(void* arg) {
  chunk_pool* pool = (chunk_pool*)arg;
  for (;;) {
    const uint64_t c = atomic_fetch_add_explicit(&pool->next, 1, memory_order_relaxed);
    if (c >= pool->count) return NULL;
    pool->fn(pool->ctx, c);
  }
}

static int hardware_threads(void) {
  long hc = 0;
#ifdef _SC_NPROCESSORS_ONLN
  hc = sysconf(_SC_NPROCESSORS_ONLN);
#endif
  return hc > 0 ? (int)hc : 1;
}

static void parallel_chunks(uint64_t count, int threads, chunk_fn fn, void* ctx) {
  if (count == 0) return;
  uint64_t workers = (uint64_t)(threads > 0 ? threads : hardware_threads());
  if (workers > count) workers = count;
  if (workers <= 1) {
    for (uint64_t c = 0; c < count; ++c) fn(ctx, c);
    return;
  }
  chunk_pool pool;
  atomic_init(&pool.next, 0);
  pool.count = count;
  pool.fn = fn;
  pool.ctx = ctx;
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (workers - 1));
  for (uint64_t w = 1; w < workers; ++w) pthread_create(&tids[w - 1], NULL, chunk_worker, &pool);
  chunk_worker(&pool);
  for (uint64_t w = 1; w < workers; ++w) pthread_join(tids[w - 1], NULL);
  free(tids);
}

/* ------------------------------------------------------------------ jl.cpp */

/* proj/src/jl.cpp:13-36 */
int or_sample_jl(int64_t k, int64_t d, uint64_t seed, double* out) {
  if (k < 1 || d < 1) return -1;
  const double scale = 1.0 / sqrt((double)k);
  for (int64_t i = 0; i < k; ++i)
    for (int64_t j = 0; j < d; ++j)
      out[i * d + j] = scale * or_rademacher_sign(seed, (uint64_t)i, (uint64_t)j);
  return 0;
}

/* proj/src/jl.cpp:38-50 */
int64_t or_jl_dimension(int64_t n_points, double epsilon, double gamma) {
  if (n_points < 2) return -1;
  if (!(epsilon > 0.0 && epsilon < 1.0)) return -1;
  if (!(gamma > 0.0 && gamma < 1.0)) return -1;
  const double n = (double)n_points;
  const double denom = epsilon * epsilon / 2.0 - epsilon * epsilon * epsilon / 3.0;
  const double k = 4.0 * log(n * n / gamma) / denom;
  return (int64_t)ceil(k);
}

/* ------------------------------------------------------------- dataset.cpp */

/* proj/src/dataset.cpp:209-216 (Eigen colwise().mean(): sum / n). */
void or_center(const double* X, int64_t n, int64_t d, double* mean, double* centered) {
  for (int64_t j = 0; j < d; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += X[i * d + j];
    mean[j] = acc / (double)n;
  }
  if (centered)
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < d; ++j) centered[i * d + j] = X[i * d + j] - mean[j];
}

/* --------------------------------------------------------------- embed.cpp */

typedef struct {
  const double *mean, *P, *S, *X;
  int64_t s, k, d, n;
  double* out;
} transform_ctx;

/* proj/src/embed.cpp:143-159, one row. */
static void transform_row(const transform_ctx* t, int64_t row, double* c, double* coords) {
  const int64_t d = t->d, s = t->s, k = t->k;
  const double* w = t->X + row * d;
  double* o = t->out + row * (s + k);
  for (int64_t j = 0; j < d; ++j) c[j] = w[j] - t->mean[j];
  if (s > 0) {
    for (int64_t a = 0; a < s; ++a) {
      double acc = 0.0;
      for (int64_t j = 0; j < d; ++j) acc += t->P[a * d + j] * c[j];
      coords[a] = acc;
      o[a] = acc;
    }
    /* residual = c - P^T coords */
    for (int64_t j = 0; j < d; ++j) {
      double acc = 0.0;
      for (int64_t a = 0; a < s; ++a) acc += t->P[a * d + j] * coords[a];
      c[j] -= acc;
    }
  }
  for (int64_t b = 0; b < k; ++b) {
    double acc = 0.0;
    for (int64_t j = 0; j < d; ++j) acc += t->S[b * d + j] * c[j];
    o[s + b] = acc;
  }
}

/* proj/src/embed.cpp:170-179: 32-row chunks. */
static void transform_chunk(void* ctx, uint64_t chunk) {
  transform_ctx* t = (transform_ctx*)ctx;
  const int64_t begin = (int64_t)chunk * 32;
  int64_t end = begin + 32;
  if (end > t->n) end = t->n;
  double* c = (double*)malloc(sizeof(double) * (size_t)(t->d + t->s + 1));
  double* coords = c + t->d;
  for (int64_t i = begin; i < end; ++i) transform_row(t, i, c, coords);
  free(c);
}

void or_transform_all(const double* mean, const double* P, int64_t s, const double* S,
                      int64_t k, int64_t d, const double* X, int64_t n, double* out,
                      int threads) {
  transform_ctx t = {mean, P, S, X, s, k, d, n, out};
  parallel_chunks((uint64_t)((n + 31) / 32), threads, transform_chunk, &t);
}

/* ---------------------------------------------------------- distortion.cpp */

/* proj/src/distortion.cpp:19-34 (Neumaier). */
typedef struct {
  double sum, compensation;
} comp_sum;

static void comp_add(comp_sum* c, double value) {
  const double t = c->sum + value;
  if (fabs(c->sum) >= fabs(value))
    c->compensation += (c->sum - t) + value;
  else
    c->compensation += (value - t) + c->sum;
  c->sum = t;
}
static double comp_total(const comp_sum* c) { return c->sum + c->compensation; }

/* proj/src/distortion.cpp:46-57 */
void or_decode_pair(uint64_t p, uint64_t n, uint64_t* i_out, uint64_t* j_out) {
  const double nn = (double)n;
  double guess =
      floor((2.0 * nn - 1.0 - sqrt((2.0 * nn - 1.0) * (2.0 * nn - 1.0) - 8.0 * (double)p)) / 2.0);
  if (guess < 0.0) guess = 0.0;
  uint64_t i = (uint64_t)guess;
#define ROW_START(r) ((r) * (2 * n - (r) - 1) / 2)
  while (i > 0 && ROW_START(i) > p) --i;
  while (ROW_START(i + 1) <= p) ++i;
  *i_out = i;
  *j_out = i + 1 + (p - ROW_START(i));
#undef ROW_START
}

/* Floyd's algorithm, proj/src/distortion.cpp:90-103.  The reference's
 * std::unordered_set only affects iteration order, which the final sort
 * removes; an open-addressing set is equivalent. */
typedef struct {
  uint64_t* keys;
  uint8_t* used;
  uint64_t mask;
} u64_set;

static int set_insert(u64_set* s, uint64_t v) {
  uint64_t h = or_mix64(v) & s->mask;
  while (s->used[h]) {
    if (s->keys[h] == v) return 0;
    h = (h + 1) & s->mask;
  }
  s->used[h] = 1;
  s->keys[h] = v;
  return 1;
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int or_sample_pair_indices(uint64_t total, uint64_t m, uint64_t seed, uint64_t* out) {
  if (m < 1 || m > total) return -1;
  uint64_t cap = 16;
  while (cap < 2 * m + 2) cap <<= 1;
  u64_set set = {(uint64_t*)malloc(sizeof(uint64_t) * cap), (uint8_t*)calloc(cap, 1), cap - 1};
  seeded_rng rng;
  rng_init(&rng, seed);
  for (uint64_t t = total - m; t < total; ++t) {
    const uint64_t v = rng_below(&rng, t + 1);
    if (!set_insert(&set, v)) set_insert(&set, t);
  }
  uint64_t c = 0;
  for (uint64_t h = 0; h < cap; ++h)
    if (set.used[h]) out[c++] = set.keys[h];
  free(set.keys);
  free(set.used);
  qsort(out, (size_t)m, sizeof(uint64_t), cmp_u64);
  return 0;
}

/* proj/src/distortion.cpp:107-111 */
double or_pair_distortion(const double* x, const double* y, const double* fx, const double* fy,
                          int64_t d, int64_t r) {
  double o = 0.0, e = 0.0;
  for (int64_t t = 0; t < d; ++t) o += (x[t] - y[t]) * (x[t] - y[t]);
  for (int64_t t = 0; t < r; ++t) e += (fx[t] - fy[t]) * (fx[t] - fy[t]);
  const double orig = sqrt(o);
  if (orig == 0.0) return -1.0;
  return fabs(sqrt(e) / orig - 1.0);
}

/* Row access for fp64 or fp32 storage (fp32 widened exactly). */
typedef struct {
  const void* orig;
  const void* emb;
  int is_f32;
  int64_t d, r;
} cloud_pair;

/* proj/src/distortion.cpp:59-75: direct differences, zero rule at :66-69,
 * formula at :74. */
static double pair_value(const cloud_pair* c, uint64_t i, uint64_t j, int* zero) {
  const int64_t d = c->d, r = c->r;
  double orig_sq = 0.0, emb_sq = 0.0;
  if (c->is_f32) {
    const float* xi = (const float*)c->orig + i * d;
    const float* xj = (const float*)c->orig + j * d;
    for (int64_t t = 0; t < d; ++t) {
      const double df = (double)xi[t] - (double)xj[t];
      orig_sq += df * df;
    }
  } else {
    const double* xi = (const double*)c->orig + i * d;
    const double* xj = (const double*)c->orig + j * d;
    for (int64_t t = 0; t < d; ++t) {
      const double df = xi[t] - xj[t];
      orig_sq += df * df;
    }
  }
  if (orig_sq == 0.0) {
    *zero = 1;
    return 0.0;
  }
  *zero = 0;
  if (c->is_f32) {
    const float* fi = (const float*)c->emb + i * r;
    const float* fj = (const float*)c->emb + j * r;
    for (int64_t t = 0; t < r; ++t) {
      const double df = (double)fi[t] - (double)fj[t];
      emb_sq += df * df;
    }
  } else {
    const double* fi = (const double*)c->emb + i * r;
    const double* fj = (const double*)c->emb + j * r;
    for (int64_t t = 0; t < r; ++t) {
      const double df = fi[t] - fj[t];
      emb_sq += df * df;
    }
  }
  return fabs(sqrt(emb_sq) / sqrt(orig_sq) - 1.0);
}

/* BlockStats, proj/src/distortion.cpp:36-42, plus the argmax extension. */
typedef struct {
  double max;
  uint64_t argp; /* lowest linear pair index attaining max */
  int has_arg;
  comp_sum sum;
  uint64_t evaluated, zero_pairs;
  uint64_t* histogram; /* hist_bins + 1 */
  uint64_t* edge_near; /* hist_bins, optional */
} block_stats;

typedef struct {
  cloud_pair cloud;
  uint64_t n, p_begin, p_end, ppb;
  int all_pairs;
  const uint64_t* sampled;
  int hist_bins;
  double hist_max, edge_band;
  block_stats* blocks;
} eval_ctx;

/* proj/src/distortion.cpp:77-88 (record) with argmax tracking. */
static void record(const eval_ctx* e, block_stats* st, double value, uint64_t p) {
  if (!st->has_arg || value > st->max) {
    st->max = value;
    st->argp = p;
    st->has_arg = 1;
  }
  comp_add(&st->sum, value);
  ++st->evaluated;
  if (value >= e->hist_max) {
    ++st->histogram[e->hist_bins];
  } else {
    uint64_t bin = (uint64_t)(value / e->hist_max * e->hist_bins);
    if (bin > (uint64_t)(e->hist_bins - 1)) bin = (uint64_t)(e->hist_bins - 1);
    ++st->histogram[bin];
  }
  if (st->edge_near) {
    const double w = e->hist_max / e->hist_bins;
    const double pos = value / w;
    long kk = lround(pos);
    for (long q = kk - 1; q <= kk + 1; ++q) {
      if (q < 1 || q > e->hist_bins) continue;
      const double dist = fabs(value - (double)q * w);
      if (dist <= e->edge_band) ++st->edge_near[q - 1];
      if (dist <= 10.0 * e->edge_band) ++st->edge_near[e->hist_bins + q - 1];
    }
  }
}

/* proj/src/distortion.cpp:143-169: one block. */
static void eval_block(void* ctx, uint64_t b) {
  eval_ctx* e = (eval_ctx*)ctx;
  block_stats* st = &e->blocks[b];
  const uint64_t begin = e->p_begin + b * e->ppb;
  uint64_t end = begin + e->ppb;
  if (end > e->p_end) end = e->p_end;
  uint64_t i = 0, j = 0;
  if (e->all_pairs && begin < end) or_decode_pair(begin, e->n, &i, &j);
  for (uint64_t p = begin; p < end; ++p) {
    uint64_t pid = p;
    if (!e->all_pairs) {
      pid = e->sampled[p];
      or_decode_pair(pid, e->n, &i, &j);
    } else if (p != begin) {
      if (++j >= e->n) {
        ++i;
        j = i + 1;
      }
    }
    int zero = 0;
    const double value = pair_value(&e->cloud, i, j, &zero);
    if (zero)
      ++st->zero_pairs;
    else
      record(e, st, value, pid);
  }
}

static int evaluate_impl(const cloud_pair* cloud, int64_t n, int all_pairs, uint64_t m,
                         uint64_t sample_seed, int hist_bins, double hist_max,
                         uint64_t pairs_per_block, int threads, or_report* rep, uint64_t* hist,
                         double edge_band, uint64_t* edge_near, int64_t row_begin,
                         int64_t row_end) {
  /* proj/src/distortion.cpp:116-134: validation. */
  if (hist_bins < 1 || !(hist_max > 0.0)) return -1;
  if (pairs_per_block == 0) pairs_per_block = 1;
  const uint64_t un = (uint64_t)n;
  const uint64_t total_pairs = un * (un - 1) / 2;
  uint64_t* sampled = NULL;
  uint64_t p_begin = 0, p_end = total_pairs;
  if (!all_pairs) {
    if (m < 1 || m > total_pairs) return -1;
    sampled = (uint64_t*)malloc(sizeof(uint64_t) * m);
    or_sample_pair_indices(total_pairs, m, sample_seed, sampled);
    p_end = m;
  } else {
    if (row_begin < 0) row_begin = 0;
    if (row_end > n) row_end = n;
    const uint64_t rb = (uint64_t)row_begin, re = (uint64_t)row_end;
    p_begin = rb * (2 * un - rb - 1) / 2;
    p_end = re >= un ? total_pairs : re * (2 * un - re - 1) / 2;
    if (p_end < p_begin) p_end = p_begin;
  }
  const uint64_t work = p_end - p_begin;
  const uint64_t n_blocks = work == 0 ? 0 : (work + pairs_per_block - 1) / pairs_per_block;
  block_stats* blocks = (block_stats*)calloc(n_blocks ? n_blocks : 1, sizeof(block_stats));
  const uint64_t hb = (uint64_t)hist_bins + 1;
  uint64_t* hstore = (uint64_t*)calloc((n_blocks ? n_blocks : 1) * hb, sizeof(uint64_t));
  uint64_t* estore =
      edge_band > 0.0 ? (uint64_t*)calloc((n_blocks ? n_blocks : 1) * 2 * (hb - 1), sizeof(uint64_t))
                      : NULL;
  for (uint64_t b = 0; b < n_blocks; ++b) {
    blocks[b].histogram = hstore + b * hb;
    blocks[b].edge_near = estore ? estore + b * 2 * (hb - 1) : NULL;
  }
  eval_ctx e = {*cloud, un,          p_begin,   p_end,     pairs_per_block, all_pairs,
                sampled, hist_bins, hist_max, edge_band, blocks};
  parallel_chunks(n_blocks, threads, eval_block, &e);

  /* Ordered merge, proj/src/distortion.cpp:176-190. */
  memset(rep, 0, sizeof(*rep));
  rep->hist_bins = hist_bins;
  rep->hist_max = hist_max;
  rep->sampled = !all_pairs;
  rep->sample_seed = all_pairs ? 0 : sample_seed;
  rep->argmax_i = rep->argmax_j = UINT64_MAX;
  memset(hist, 0, sizeof(uint64_t) * hb);
  if (edge_near) memset(edge_near, 0, sizeof(uint64_t) * 2 * (hb - 1));
  comp_sum total = {0.0, 0.0};
  int has_arg = 0;
  uint64_t argp = 0;
  double best = 0.0;
  for (uint64_t b = 0; b < n_blocks; ++b) {
    const block_stats* st = &blocks[b];
    if (st->has_arg && (!has_arg || st->max > best)) {
      best = st->max;
      argp = st->argp;
      has_arg = 1;
    }
    comp_add(&total, comp_total(&st->sum));
    rep->n_pairs_evaluated += st->evaluated;
    rep->n_zero_distance_pairs += st->zero_pairs;
    for (uint64_t k = 0; k < hb; ++k) hist[k] += st->histogram[k];
    if (edge_near && st->edge_near)
      for (uint64_t k = 0; k < 2 * (hb - 1); ++k) edge_near[k] += st->edge_near[k];
  }
  rep->max_distortion = has_arg ? best : 0.0;
  if (has_arg) or_decode_pair(argp, un, &rep->argmax_i, &rep->argmax_j);
  rep->mean_distortion =
      rep->n_pairs_evaluated == 0 ? 0.0 : comp_total(&total) / (double)rep->n_pairs_evaluated;
  free(blocks);
  free(hstore);
  free(estore);
  free(sampled);
  return 0;
}

int or_evaluate(const double* orig, int64_t n, int64_t d, const double* emb, int64_t n_emb,
                int64_t r, int all_pairs, uint64_t m, uint64_t sample_seed, int hist_bins,
                double hist_max, uint64_t pairs_per_block, int threads, or_report* rep,
                uint64_t* hist, double edge_band, uint64_t* edge_near, int64_t row_begin,
                int64_t row_end) {
  if (n != n_emb) return -1; /* distortion.cpp:116-119 */
  cloud_pair c = {orig, emb, 0, d, r};
  return evaluate_impl(&c, n, all_pairs, m, sample_seed, hist_bins, hist_max, pairs_per_block,
                       threads, rep, hist, edge_band, edge_near, row_begin, row_end);
}

int or_evaluate_f32(const float* orig, int64_t n, int64_t d, const float* emb, int64_t r,
                    int hist_bins, double hist_max, int threads, or_report* rep, uint64_t* hist,
                    int64_t row_begin, int64_t row_end) {
  cloud_pair c = {orig, emb, 1, d, r};
  return evaluate_impl(&c, n, 1, 0, 0, hist_bins, hist_max, 16384, threads, rep, hist, 0.0,
                       NULL, row_begin, row_end);
}

/* Sampled mode (proj/src/distortion.cpp:90-103, :151-154) on fp32 clouds. */
int or_evaluate_f32_sampled(const float* orig, int64_t n, int64_t d, const float* emb, int64_t r,
                            uint64_t m, uint64_t sample_seed, int hist_bins, double hist_max,
                            int threads, or_report* rep, uint64_t* hist) {
  cloud_pair c = {orig, emb, 1, d, r};
  return evaluate_impl(&c, n, 0, m, sample_seed, hist_bins, hist_max, 16384, threads, rep, hist, 0.0,
                       NULL, 0, n);
}

/* proj/tests/test_util.hpp:57-84 */
void or_naive_distortion(const double* orig, int64_t n, int64_t d, const double* emb, int64_t r,
                         double* max_out, double* mean_out, uint64_t* evaluated,
                         uint64_t* zero_pairs) {
  double mx = 0.0;
  long double sum = 0.0L;
  uint64_t ev = 0, zp = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = i + 1; j < n; ++j) {
      double o = 0.0, e = 0.0;
      for (int64_t t = 0; t < d; ++t) o += (orig[i * d + t] - orig[j * d + t]) * (orig[i * d + t] - orig[j * d + t]);
      const double on = sqrt(o);
      if (on == 0.0) {
        ++zp;
        continue;
      }
      for (int64_t t = 0; t < r; ++t) e += (emb[i * r + t] - emb[j * r + t]) * (emb[i * r + t] - emb[j * r + t]);
      const double value = fabs(sqrt(e) / on - 1.0);
      if (value > mx) mx = value;
      sum += value;
      ++ev;
    }
  }
  *max_out = mx;
  *mean_out = ev == 0 ? 0.0 : (double)(sum / ev);
  *evaluated = ev;
  *zero_pairs = zp;
}

/* ------------------------------------------------- screen error-band counts
 * TEST INFRASTRUCTURE for the GPU SCREEN engine's histogram (not a reference
 * function).  For every pair i<j of fp32 clouds, the exact value v (the
 * reference formula above) and the screen's rigorous per-pair error bound
 *   t = rel_eps (sn/o + sm/e)(1 + v),
 * sn = nx[i] + nx[j], sm = ny[i] + ny[j] (squared norms of the rows after the
 * screen's centring shift), o / e the exact squared distances.  out[q-1]
 * counts the pairs within t of edge q (q = 1..hist_bins, edge q*hist_max/bins)
 * and out[hist_bins + q-1] those within t * frac.  A screened value can only
 * leave its exact bin across an edge it lies within t of. */
typedef struct {
  const float *x, *y;
  const double *nx, *ny;
  int64_t n, d, r;
  double rel_eps, frac, hist_max;
  int bins;
  uint64_t* part; /* per row block: 2 * bins */
  int64_t rows_per;
} band_ctx;

static void band_block(void* vctx, uint64_t b) {
  band_ctx* c = (band_ctx*)vctx;
  uint64_t* out = c->part + b * 2 * (uint64_t)c->bins;
  const double w = c->hist_max / c->bins;
  const int64_t i0 = (int64_t)b * c->rows_per;
  const int64_t i1 = i0 + c->rows_per < c->n ? i0 + c->rows_per : c->n;
  for (int64_t i = i0; i < i1; ++i) {
    const float* xi = c->x + i * c->d;
    const float* fi = c->y + i * c->r;
    for (int64_t j = i + 1; j < c->n; ++j) {
      const float* xj = c->x + j * c->d;
      const float* fj = c->y + j * c->r;
      double o = 0.0, e = 0.0;
      for (int64_t t = 0; t < c->d; ++t) {
        const double df = (double)xi[t] - (double)xj[t];
        o += df * df;
      }
      if (o == 0.0) continue;
      for (int64_t t = 0; t < c->r; ++t) {
        const double df = (double)fi[t] - (double)fj[t];
        e += df * df;
      }
      const double v = fabs(sqrt(e) / sqrt(o) - 1.0);
      const double tb = c->rel_eps * ((c->nx[i] + c->nx[j]) / o +
                                      (e > 0.0 ? (c->ny[i] + c->ny[j]) / e : 1e300)) * (1.0 + v);
      const long kk = lround(v / w);
      for (long q = kk - 1; q <= kk + 1; ++q) {
        if (q < 1 || q > c->bins) continue;
        const double dist = fabs(v - (double)q * w);
        if (dist <= tb) ++out[q - 1];
        if (dist <= tb * c->frac) ++out[c->bins + q - 1];
      }
    }
  }
}

int or_edge_band_counts(const float* x, const float* y, int64_t n, int64_t d, int64_t r,
                        const double* nx, const double* ny, double rel_eps, double frac,
                        int hist_bins, double hist_max, int threads, uint64_t* out) {
  if (hist_bins < 1 || !(hist_max > 0.0) || n < 0) return -1;
  const int64_t rows_per = 16;
  const uint64_t blocks = (uint64_t)((n + rows_per - 1) / rows_per);
  uint64_t* part = (uint64_t*)calloc((blocks ? blocks : 1) * 2 * (uint64_t)hist_bins, sizeof(uint64_t));
  band_ctx c = {x, y, nx, ny, n, d, r, rel_eps, frac, hist_max, hist_bins, part, rows_per};
  parallel_chunks(blocks, threads, band_block, &c);
  memset(out, 0, sizeof(uint64_t) * 2 * (size_t)hist_bins);
  for (uint64_t b = 0; b < blocks; ++b)
    for (int k = 0; k < 2 * hist_bins; ++k) out[k] += part[b * 2 * (uint64_t)hist_bins + k];
  free(part);
  return 0;
}

