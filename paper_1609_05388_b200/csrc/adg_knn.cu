// adg_knn.cu -- brute-force k nearest neighbours and the k-NN graph
// (proj/src/downstream.cpp:24-137) on the GPU.
//
// The reference computes, per query, every database distance as the fp64
// Euclidean norm of the row difference and keeps the k smallest (distance,
// index) pairs -- ties toward the smaller index (partial_sort on pairs,
// downstream.cpp:24-40).  Here one CTA takes 64 queries and streams the
// database through shared memory in 64-row tiles: 4 x 4 fp64 direct-
// difference accumulators per thread (no Gram form, so no cancellation --
// the same arithmetic as the reference up to summation order), then each
// warp folds its queries' 64 new candidates into per-query sorted top-k lists
// (shared memory for k <= 128, else a global scratch) behind a running k-th
// distance threshold, so after the first tiles almost every candidate is
// rejected with one compare.  The key is (sqrt(d2), index): sqrt is
// correctly rounded in fp64, as Eigen's norm(), so two squared distances that
// round to the same norm tie-break by index exactly as in the reference.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <map>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thread>

#include "adg_embed.cuh"
#include "adg_internal.cuh"
#include "adg_screen.cuh"

namespace adg {
namespace {

constexpr int KQ = 64;      // queries per CTA
constexpr int KD = 64;      // database rows per tile
constexpr int KC = 16;      // dimensions per shared-memory chunk
constexpr int KT = 256;     // threads
constexpr int KPAD = KQ + 1;

struct Cand {
  double dist;
  int64_t idx;
};

__device__ __forceinline__ bool cand_less(double d1, int64_t i1, double d2, int64_t i2) {
  return d1 < d2 || (d1 == d2 && i1 < i2);
}

template <typename TD, typename TQ>
__global__ void __launch_bounds__(KT)
knn_kernel(const TD* __restrict__ D, int64_t n, int64_t d, const TQ* __restrict__ Q, int64_t nq,
           int k, int skip_self, Cand* __restrict__ gl_lists, Cand* __restrict__ out) {
  extern __shared__ double ksm[];
  double* qs = ksm;                        // [KC][KPAD]
  double* ds = qs + KC * KPAD;             // [KC][KPAD]
  double* dt = ds + KC * KPAD;             // [KQ][KD + 1] squared distances of the tile
  double* thr_d = dt + KQ * (KD + 1);      // [KQ] k-th distance (or +inf)
  int64_t* thr_i = reinterpret_cast<int64_t*>(thr_d + KQ);  // [KQ]
  int* fill = reinterpret_cast<int*>(thr_i + KQ);           // [KQ] list sizes
  Cand* lists = gl_lists ? gl_lists + (int64_t)blockIdx.x * KQ * k
                         : reinterpret_cast<Cand*>(fill + KQ + (KQ & 1));
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int tq = tid / 16, td = tid % 16;
  const int64_t q0 = (int64_t)blockIdx.x * KQ;
  for (int q = tid; q < KQ; q += KT) {
    thr_d[q] = INFINITY;
    thr_i[q] = INT64_MAX;
    fill[q] = 0;
  }
  __syncthreads();
  for (int64_t j0 = 0; j0 < n; j0 += KD) {
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int64_t c0 = 0; c0 < d; c0 += KC) {
      for (int e = tid; e < KQ * KC; e += KT) {
        const int q = e / KC, c = e % KC;
        const int64_t gq = q0 + q, gc = c0 + c;
        qs[c * KPAD + q] = (gq < nq && gc < d) ? to_f64(Q[gq * d + gc]) : 0.0;
      }
      for (int e = tid; e < KD * KC; e += KT) {
        const int j = e / KC, c = e % KC;
        const int64_t gj = j0 + j, gc = c0 + c;
        ds[c * KPAD + j] = (gj < n && gc < d) ? to_f64(D[gj * d + gc]) : 0.0;
      }
      __syncthreads();
#pragma unroll 4
      for (int c = 0; c < KC; ++c) {
        double qv[4], dv[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) qv[a] = qs[c * KPAD + tq + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) dv[b] = ds[c * KPAD + td + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const double df = dv[b] - qv[a];  // row_i - query, as downstream.cpp:30
            acc[a][b] = fma(df, df, acc[a][b]);
          }
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dt[(tq + 16 * a) * (KD + 1) + td + 16 * b] = acc[a][b];
    __syncthreads();
    // fold the tile's candidates into each query's sorted top-k list
    for (int q = warp; q < KQ; q += KT / 32) {
      const int64_t gq = q0 + q;
      if (gq >= nq) continue;
      Cand* L = lists + (int64_t)q * k;
#pragma unroll
      for (int h = 0; h < KD / 32; ++h) {
        const int c = h * 32 + lane;
        const int64_t j = j0 + c;
        double dist = INFINITY;
        bool ok = j < n && !(skip_self && j == gq);
        const double s2 = dt[q * (KD + 1) + c];
        // s2 > thr^2 (1 + 1e-12) implies sqrt(s2) > thr strictly: reject
        // without the fp64 sqrt (almost every candidate once the list is full)
        const double td = thr_d[q];
        ok = ok && !(s2 > td * td * (1.0 + 1e-12));
        if (ok) dist = sqrt(s2);
        ok = ok && cand_less(dist, j, td, thr_i[q]);
        unsigned pend = __ballot_sync(0xffffffffu, ok);
        while (pend) {
          const int src = __ffs(pend) - 1;
          pend &= pend - 1;
          const double cd = __shfl_sync(0xffffffffu, dist, src);
          const int64_t ci = __shfl_sync(0xffffffffu, j, src);
          const int m = fill[q];
          if (!cand_less(cd, ci, thr_d[q], thr_i[q])) continue;  // threshold moved
          // position = number of entries smaller than the candidate
          int pos = 0;
          for (int b = lane; b < m; b += 32) pos += cand_less(L[b].dist, L[b].idx, cd, ci) ? 1 : 0;
          for (int s = 16; s; s >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, s);
          const int last = m < k ? m : k - 1;  // entries [pos, last) move one slot right
          for (int b0 = pos; b0 < last; b0 += 32) {
            const int b = last - 1 - (b0 - pos) - lane;  // from the end, 32 at a time
            Cand v;
            const bool mv = b >= pos;
            if (mv) v = L[b];
            __syncwarp();
            if (mv) L[b + 1] = v;
            __syncwarp();
          }
          if (lane == 0) {
            L[pos] = Cand{cd, ci};
            const int nm = m < k ? m + 1 : k;
            fill[q] = nm;
            if (nm == k) {
              thr_d[q] = L[k - 1].dist;
              thr_i[q] = L[k - 1].idx;
            }
          }
          __syncwarp();
        }
      }
    }
    __syncthreads();
  }
  // sorted lists out
  for (int e = tid; e < KQ * k; e += KT) {
    const int q = e / k, b = e % k;
    const int64_t gq = q0 + q;
    if (gq < nq) out[gq * k + b] = b < fill[q] ? lists[(int64_t)q * k + b] : Cand{INFINITY, -1};
  }
}

// all_lists (nq x k, device): each query's k nearest database rows, ascending.
void knn_device(adg_ctx* ctx, const void* D, adg_dtype dd, int64_t n, int64_t d, const void* Q,
                adg_dtype qd, int64_t nq, int k, bool skip_self, Cand* all_lists) {
  if (nq == 0) return;
  const size_t fixed = sizeof(double) * (size_t)(2 * KC * KPAD + KQ * (KD + 1) + 2 * KQ) +
                       sizeof(int) * (KQ + 2);
  const size_t list_bytes = sizeof(Cand) * (size_t)KQ * (size_t)k;
  const bool in_smem = fixed + list_bytes <= 200 * 1024;
  const int64_t blocks = (nq + KQ - 1) / KQ;
  DevBuf<Cand> scratch(in_smem ? 0 : (size_t)(blocks * KQ * k), ctx->stream);
  const size_t smem = fixed + (in_smem ? list_bytes : 0);
  ADG_DISPATCH_DTYPE(dd, TD, {
    ADG_DISPATCH_DTYPE(qd, TQ, {
      auto kern = knn_kernel<TD, TQ>;
      ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<(unsigned)blocks, KT, smem, ctx->stream>>>((const TD*)D, n, d, (const TQ*)Q, nq, k,
                                                        skip_self ? 1 : 0,
                                                        in_smem ? nullptr : scratch.ptr, all_lists);
    });
  });
  after_launch(ctx);
}

// ---------------------------------------------------------------------------
// k-NN graph on the tensor cores (all rows against all rows, skip self).
//
//  1. radii: m evenly spaced sample rows; approximate distances to them by a
//     3xTF32 projection (TransformPlan with W = the centred sample rows); per
//     row the k+1 nearest by that estimate, their exact distances (the
//     refine's own fp64 formula), tau_i = the largest.  k+1 distinct rows lie
//     within tau_i, at most one of them row i itself, so the exact k-th
//     neighbour distance is <= tau_i -- whatever the estimate's error.
//  2. the split-fp16 screen (HMODE 4) appends every pair whose screened lower
//     bound reaches a side's radius, with its bracket [lo, hi] of the squared
//     distance, as a candidate of that side's row.
//  3. candidates grouped by query (count, scan, scatter); per query U = the
//     k-th smallest hi; candidates with lo > U are farther than k others and
//     dropped; the rest get the exact fp64 distance (same summation as
//     knn_kernel, so the same bits) and the k smallest (distance, index) win.
// Every true neighbour passes every filter (lo <= d*^2 <= tau^2, lo <= U), so
// the lists equal knn_kernel's exactly.
// ADG_KNN_PROFILE=1: stage wall times (synchronised) to stderr -- profiling aid
struct KnnStageTimer {
  adg_ctx* ctx;
  bool on;
  std::chrono::steady_clock::time_point t0;
  explicit KnnStageTimer(adg_ctx* c) : ctx(c), on(std::getenv("ADG_KNN_PROFILE") != nullptr) {
    if (on) {
      cudaStreamSynchronize(ctx->stream);
      t0 = std::chrono::steady_clock::now();
    }
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(ctx->stream);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[knn] %-10s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

constexpr int KNN_SAMPLE_CHUNK = 256;
constexpr int KNN_MAX_SAMPLE = 2048;
constexpr int KNN_TC_MAX_K = 64;

template <typename T>
__global__ void sample_rows_kernel(const T* __restrict__ X, int64_t n, int64_t d, int64_t m,
                                   int64_t t0, int64_t cnt, const double* __restrict__ mean,
                                   double* __restrict__ P, double* __restrict__ pn) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= cnt) return;
  const int64_t row = (t0 + w) * n / m;
  double acc = 0.0;
  for (int64_t c = lane; c < d; c += 32) {
    const double v = to_f64(X[row * d + c]) - mean[c];
    P[w * d + c] = v;
    acc = fma(v, v, acc);
  }
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) pn[t0 + w] = acc;
}

template <typename T>
__global__ void centred_norm_kernel(const T* __restrict__ X, int64_t n, int64_t d,
                                    const double* __restrict__ mean, float* __restrict__ xn) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double acc = 0.0;
  for (int64_t c = lane; c < d; c += 32) {
    const double v = to_f64(X[row * d + c]) - mean[c];
    acc = fma(v, v, acc);
  }
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) xn[row] = (float)acc;
}

__device__ __forceinline__ uint32_t fkey(float f) {  // monotone float -> uint
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// exact squared distance, knn_kernel's arithmetic: sum over c in order of
// fma(df, df, .) with df = row_j - query.  With 16-byte aligned rows a lane
// fetches 128 bytes of its row per step (8 loads in flight, each line read
// once) and then runs the same in-order FMA chain over them.
__device__ __forceinline__ void unpack16(const uint4 u, float (&v)[4]) {
  v[0] = __uint_as_float(u.x);
  v[1] = __uint_as_float(u.y);
  v[2] = __uint_as_float(u.z);
  v[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ void unpack16(const uint4 u, __nv_bfloat16 (&v)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __ushort_as_bfloat16((unsigned short)(w[i] & 0xffffu));
    v[2 * i + 1] = __ushort_as_bfloat16((unsigned short)(w[i] >> 16));
  }
}
__device__ __forceinline__ void unpack16(const uint4 u, double (&v)[2]) {
  v[0] = __hiloint2double((int)u.y, (int)u.x);
  v[1] = __hiloint2double((int)u.w, (int)u.z);
}

template <typename T>
__device__ __forceinline__ double exact_d2(const T* __restrict__ X, int64_t d, int64_t j, int64_t q,
                                           bool vec) {
  const T* a = X + j * d;
  const T* b = X + q * d;
  double acc = 0.0;
  int64_t c = 0;
  if (vec) {
    constexpr int E = 16 / (int)sizeof(T);
    const uint4* a4 = reinterpret_cast<const uint4*>(a);
    const uint4* b4 = reinterpret_cast<const uint4*>(b);
    const int64_t nv = d / E;
    int64_t v = 0;
    for (; v + 8 <= nv; v += 8) {
      uint4 ra[8], rb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        ra[u] = __ldg(a4 + v + u);
        rb[u] = __ldg(b4 + v + u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        T ea[E], eb[E];
        unpack16(ra[u], ea);
        unpack16(rb[u], eb);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double df = to_f64(ea[e]) - to_f64(eb[e]);
          acc = fma(df, df, acc);
        }
      }
    }
    for (; v < nv; ++v) {
      T ea[E], eb[E];
      unpack16(__ldg(a4 + v), ea);
      unpack16(__ldg(b4 + v), eb);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double df = to_f64(ea[e]) - to_f64(eb[e]);
        acc = fma(df, df, acc);
      }
    }
    c = nv * E;
  }
  for (; c < d; ++c) {
    const double df = to_f64(a[c]) - to_f64(b[c]);
    acc = fma(df, df, acc);
  }
  return acc;
}

// one warp per row: tau_i^2 (rounded up to fp32) from the k+1 sample rows
// nearest by the estimate
template <typename T>
__global__ void __launch_bounds__(256)
knn_radius_kernel(const T* __restrict__ X, int64_t n, int64_t d, int m, int K,
                  const float* __restrict__ G, const float* __restrict__ xn,
                  const double* __restrict__ pn, float* __restrict__ tau2, bool vec) {
  __shared__ int sel[8][KNN_TC_MAX_K + 1];
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (i >= n) return;
  constexpr int MQ = KNN_MAX_SAMPLE / 32;
  uint32_t key[MQ];
  const float xi = xn[i];
#pragma unroll
  for (int q = 0; q < MQ; ++q) {
    const int t = q * 32 + lane;
    key[q] = 0xffffffffu;
    if (t < m) {
      const int c = t / KNN_SAMPLE_CHUNK, tt = t % KNN_SAMPLE_CHUNK;
      const float g = G[((int64_t)c * n + i) * KNN_SAMPLE_CHUNK + tt];
      key[q] = fkey(fmaf(-2.0f, g, xi + (float)pn[t]));
    }
  }
  // smallest T with #{key <= T} >= K
  uint32_t lo = 0u, hi = 0xffffffffu;
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    int c = 0;
#pragma unroll
    for (int q = 0; q < MQ; ++q) c += key[q] <= mid ? 1 : 0;
    for (int s = 16; s; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (c >= K) hi = mid; else lo = mid + 1;
  }
  // the first K sample rows (in t order) with key <= T
  int taken = 0;
#pragma unroll
  for (int q = 0; q < MQ; ++q) {
    const bool ok = key[q] <= lo;
    const unsigned b = __ballot_sync(0xffffffffu, ok);
    const int pos = taken + __popc(b & ((1u << lane) - 1u));
    if (ok && pos < K) sel[wib][pos] = q * 32 + lane;
    taken += __popc(b);
  }
  __syncwarp();
  double worst = 0.0;
  for (int a = lane; a < K; a += 32) {
    const int64_t row = (int64_t)sel[wib][a] * n / m;
    worst = fmax(worst, exact_d2(X, d, row, i, vec));
  }
  for (int s = 16; s; s >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, s));
  if (lane == 0) tau2[i] = __double2float_ru(worst * (1.0 + 1e-9));
}

__global__ void knn_count_kernel(const uint4* __restrict__ E, int64_t used, uint32_t* __restrict__ cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < used;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t q = E[e].x;
    if (q != 0xffffffffu) atomicAdd(&cnt[q], 1u);
  }
}

__global__ void knn_scatter_kernel(const uint4* __restrict__ E, int64_t used,
                                   const uint32_t* __restrict__ off, uint32_t* __restrict__ cur,
                                   uint4* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < used;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = E[e];
    if (v.x == 0xffffffffu) continue;
    out[off[v.x] + atomicAdd(&cur[v.x], 1u)] = v;
  }
}

// one warp per query: prune by the k-th smallest upper bound, refine exactly,
// keep the k smallest (distance, index)
template <typename T>
__global__ void __launch_bounds__(256)
knn_select_kernel(const T* __restrict__ X, int64_t n, int64_t d, int k, bool vec,
                  const uint32_t* __restrict__ off, uint4* __restrict__ C, Cand* __restrict__ out,
                  unsigned long long* __restrict__ stat) {
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= n) return;
  const int64_t b0 = off[q], cnt = (int64_t)off[q + 1] - b0;
  uint4* L = C + b0;
  if (cnt < k) {  // cannot happen: every true neighbour is a candidate
    if (lane == 0) atomicExch(stat, 1ull);
    return;
  }
  // U = k-th smallest hi
  uint32_t lo = 0u, hi = 0xffffffffu;
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    int c = 0;
    for (int64_t a = lane; a < cnt; a += 32) c += fkey(__uint_as_float(L[a].w)) <= mid ? 1 : 0;
    for (int s = 16; s; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (c >= k) hi = mid; else lo = mid + 1;
  }
  const float U = fkey_inv(lo);
  // survivors compacted in place (writes land at or below the slots the warp
  // has already read), then their exact distances with every lane busy
  int64_t ns = 0;
  for (int64_t a0 = 0; a0 < cnt; a0 += 32) {
    const int64_t a = a0 + lane;
    uint32_t cid = 0;
    bool ok = false;
    if (a < cnt) {
      const uint4 v = L[a];
      cid = v.y;
      ok = __uint_as_float(v.z) <= U;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    __syncwarp();
    if (ok) L[ns + __popc(bal & ((1u << lane) - 1u))].x = cid;
    ns += __popc(bal);
    __syncwarp();
  }
  for (int64_t a = lane; a < ns; a += 32) {
    const uint32_t cid = L[a].x;
    const double dist = sqrt(exact_d2(X, d, (int64_t)cid, q, vec));
    const unsigned long long db = __double_as_longlong(dist);
    L[a] = make_uint4(cid, (uint32_t)db, (uint32_t)(db >> 32), 0u);
  }
  __syncwarp();
  if (lane == 0) atomicAdd(stat + 1, (unsigned long long)ns);
  if (ns < k) {
    if (lane == 0) atomicExch(stat, 2ull);
    return;
  }
  // k rounds of the warp minimum above the last pick
  double ld = -1.0;
  int64_t li = -1;
  for (int r = 0; r < k; ++r) {
    double bd = INFINITY;
    int64_t bi = INT64_MAX;
    for (int64_t a = lane; a < ns; a += 32) {
      const uint4 v = L[a];
      const double dd = __longlong_as_double((long long)(((unsigned long long)v.z << 32) | v.y));
      const int64_t ii = v.x;
      if (cand_less(ld, li, dd, ii) && cand_less(dd, ii, bd, bi)) {
        bd = dd;
        bi = ii;
      }
    }
    for (int s = 16; s; s >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, s);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, s);
      if (cand_less(od, oi, bd, bi)) {
        bd = od;
        bi = oi;
      }
    }
    if (lane == 0) out[q * k + r] = Cand{bd, bi};
    ld = bd;
    li = bi;
  }
}

// Tensor-core k-NN lists (n x k, skip self) into `lists`; false when the case
// is outside the path's range (the caller then runs knn_kernel).
bool knn_graph_tc(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d, int k,
                  Cand* lists) {
  if (std::getenv("ADG_KNN_SIMT")) return false;
  if (n < 4096 || k + 1 > KNN_TC_MAX_K || n > 65535LL * 160 || d < 1) return false;
  const int m = (int)std::min<int64_t>(KNN_MAX_SAMPLE, n / 2 / KNN_SAMPLE_CHUNK * KNN_SAMPLE_CHUNK);
  if (m < 16 * (k + 1)) return false;
  cudaStream_t st = ctx->stream;
  KnnStageTimer tm(ctx);
  const bool vec = (reinterpret_cast<uintptr_t>(X) & 15) == 0 && (d * (int64_t)dtype_size(dt)) % 16 == 0;
  // 1. radii
  DevBuf<float> tau2;
  {
    DevBuf<double> mean((size_t)d, st), P((size_t)(KNN_SAMPLE_CHUNK * d), st), pn((size_t)m, st);
    DevBuf<float> G((size_t)((int64_t)m * n), st), xn((size_t)n, st);
    column_means_sampled(ctx, X, dt, n, d, 4096, mean.ptr);
    ADG_DISPATCH_DTYPE(dt, T, {
      centred_norm_kernel<T><<<blocks_for(n * 32, 256), 256, 0, st>>>((const T*)X, n, d, mean.ptr, xn.ptr);
    });
    after_launch(ctx);
    for (int c = 0; c < m / KNN_SAMPLE_CHUNK; ++c) {
      ADG_DISPATCH_DTYPE(dt, T, {
        sample_rows_kernel<T><<<blocks_for(KNN_SAMPLE_CHUNK * 32, 256), 256, 0, st>>>(
            (const T*)X, n, d, m, (int64_t)c * KNN_SAMPLE_CHUNK, KNN_SAMPLE_CHUNK, mean.ptr, P.ptr, pn.ptr);
      });
      after_launch(ctx);
      TransformPlan plan(ctx, mean.ptr, P.ptr, KNN_SAMPLE_CHUNK, nullptr, 0, d, false);
      plan.run(X, dt, n, G.ptr + (int64_t)c * n * KNN_SAMPLE_CHUNK, ADG_F32);
    }
    tm.mark("estimate");
    const int64_t rows_pad = std::max((n + 255) / 256 * 256, (n + 159) / 160 * 160);
    tau2.alloc((size_t)rows_pad, st);
    tau2.zero();
    ADG_DISPATCH_DTYPE(dt, T, {
      knn_radius_kernel<T><<<blocks_for(n * 32, 256), 256, 0, st>>>((const T*)X, n, d, m, k + 1, G.ptr,
                                                                    xn.ptr, pn.ptr, tau2.ptr, vec);
    });
    after_launch(ctx);
    tm.mark("radii");
  }
  // 2. candidates
  ScreenOperands ops(ctx, X, dt, n, d, nullptr, ADG_F32, 0);
  tm.mark("prep");
  DevBuf<unsigned long long> count(1, st);
  long long cap = std::max<long long>(1LL << 22, (long long)(3.0 * (double)n * (k + 1) * ((double)n / m)));
  DevBuf<uint4> E;
  unsigned long long used = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    E.alloc((size_t)cap, st);
    ADG_CUDA(cudaMemsetAsync(E.ptr, 0xff, sizeof(uint4) * (size_t)cap, st));
    count.zero();
    run_screen_knn(ctx, ops, tau2.ptr, E.ptr, count.ptr, cap);
    ADG_CUDA(cudaMemcpyAsync(&used, count.ptr, sizeof(used), cudaMemcpyDeviceToHost, st));
    ADG_CUDA(cudaStreamSynchronize(st));
    tm.mark("screen");
    if ((long long)used <= cap) break;
    // second pass with room for everything, within a quarter of free memory
    size_t fr = 0, tot = 0;
    ADG_CUDA(cudaMemGetInfo(&fr, &tot));
    const long long want = (long long)(used + used / 8 + 4096);
    if ((double)want * 2 * sizeof(uint4) > 0.25 * (double)fr || attempt == 1) return false;
    cap = want;
  }
  // 3. group by query, prune, refine, select
  DevBuf<uint32_t> cntq((size_t)n + 1, st), offq((size_t)n + 1, st), cur((size_t)n, st);
  cntq.zero();
  cur.zero();
  knn_count_kernel<<<blocks_for((int64_t)used, 256), 256, 0, st>>>(E.ptr, (int64_t)used, cntq.ptr);
  after_launch(ctx);
  size_t tmp_bytes = 0;
  ADG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cntq.ptr, offq.ptr, (int)(n + 1), st));
  DevBuf<uint8_t> tmp(tmp_bytes, st);
  ADG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, tmp_bytes, cntq.ptr, offq.ptr, (int)(n + 1), st));
  uint32_t total = 0;
  ADG_CUDA(cudaMemcpyAsync(&total, offq.ptr + n, sizeof(total), cudaMemcpyDeviceToHost, st));
  ADG_CUDA(cudaStreamSynchronize(st));
  DevBuf<uint4> grouped((size_t)std::max<uint32_t>(total, 1), st);
  knn_scatter_kernel<<<blocks_for((int64_t)used, 256), 256, 0, st>>>(E.ptr, (int64_t)used, offq.ptr,
                                                                     cur.ptr, grouped.ptr);
  after_launch(ctx);
  E.release();
  tm.mark("group");
  DevBuf<unsigned long long> err(2, st);  // [error code, survivors]
  err.zero();
  ADG_DISPATCH_DTYPE(dt, T, {
    knn_select_kernel<T><<<blocks_for(n * 32, 256), 256, 0, st>>>((const T*)X, n, d, k, vec, offq.ptr,
                                                                  grouped.ptr, lists, err.ptr);
  });
  after_launch(ctx);
  unsigned long long hs[2] = {0, 0};
  ADG_CUDA(cudaMemcpyAsync(hs, err.ptr, sizeof(hs), cudaMemcpyDeviceToHost, st));
  ADG_CUDA(cudaStreamSynchronize(st));
  tm.mark("select");
  if (std::getenv("ADG_KNN_PROFILE"))
    std::fprintf(stderr, "[knn] m=%d candidates=%llu (%.1f per row) grouped=%u survivors=%.1f per row\n",
                 m, used, (double)used / (double)n, total, (double)hs[1] / (double)n);
  if (hs[0]) fail(ADG_ECUDA, "build_knn_graph: candidate set lost a neighbour (code " +
                                   std::to_string(hs[0]) + ")");
  return true;
}

// graph assembly: key (min(u, v) << 32 | max(u, v)) and distance per list entry
__global__ void edge_keys_kernel(const Cand* __restrict__ lists, int64_t n, int k,
                                 unsigned long long* __restrict__ keys, double* __restrict__ dist) {
  const int64_t N = n * k;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = t / k;
    const Cand c = lists[t];
    const unsigned long long a = (unsigned long long)(u < c.idx ? u : c.idx);
    const unsigned long long b = (unsigned long long)(u < c.idx ? c.idx : u);
    keys[t] = (a << 32) | b;
    dist[t] = c.dist;
  }
}

std::vector<Cand> knn_host(adg_ctx* ctx, const void* D, adg_dtype dd, int64_t n, int64_t d,
                           const void* Q, adg_dtype qd, int64_t nq, int k, bool skip_self) {
  ctx->last_knn_engine = 1;
  In db(D, (size_t)(n * d) * dtype_size(dd), ctx->stream);
  In qq(Q, (size_t)(nq * d) * dtype_size(qd), ctx->stream);
  DevBuf<Cand> lists((size_t)(nq * k), ctx->stream);
  knn_device(ctx, db.dev, dd, n, d, qq.dev, qd, nq, k, skip_self, lists.ptr);
  std::vector<Cand> host((size_t)(nq * k));
  if (!host.empty())
    ADG_CUDA(cudaMemcpyAsync(host.data(), lists.ptr, host.size() * sizeof(Cand),
                             cudaMemcpyDeviceToHost, ctx->stream));
  ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  return host;
}

}  // namespace
}  // namespace adg

using namespace adg;

extern "C" {

// proj/src/downstream.cpp:49-60 (knn_query) for nq queries at once.
adg_status adg_knn_query(adg_ctx* ctx, const void* database, adg_dtype dtype, int64_t n, int64_t d,
                         const void* queries, adg_dtype qdtype, int64_t nq, int64_t qdim, int k,
                         int64_t* idx_out, double* dist_out) {
  return guard_call([&] {
    ADG_REQUIRE(ctx, "null adg_ctx");
    ADG_CUDA(cudaSetDevice(ctx->device));
    if (k < 1 || k > n)
      fail(ADG_EINVAL, "knn_query: k = " + std::to_string(k) + " outside [1, " + std::to_string(n) + "]");
    if (qdim != d) fail(ADG_EINVAL, "knn_query: query dimension mismatch");
    ADG_REQUIRE(nq >= 0 && idx_out && dist_out, "knn_query: bad output");
    const std::vector<Cand> h = knn_host(ctx, database, dtype, n, d, queries, qdtype, nq, k, false);
    for (size_t t = 0; t < h.size(); ++t) {
      idx_out[t] = h[t].idx;
      dist_out[t] = h[t].dist;
    }
  });
}

// proj/src/downstream.cpp:62-88 (majority_classify)
adg_status adg_majority_classify(adg_ctx* ctx, const void* queries, adg_dtype qdtype, int64_t nq,
                                 int64_t qdim, const void* database, adg_dtype dtype, int64_t n,
                                 int64_t d, const int32_t* labels, int k, uint64_t tie_seed,
                                 int32_t* label_out) {
  return guard_call([&] {
    ADG_REQUIRE(ctx && label_out, "majority_classify: null argument");
    ADG_CUDA(cudaSetDevice(ctx->device));
    if (!labels) fail(ADG_EINVAL, "majority_classify: database has no labels");
    if (nq == 0) fail(ADG_EINVAL, "majority_classify: no query descriptors");
    if (k < 1 || k > n)
      fail(ADG_EINVAL, "knn_query: k = " + std::to_string(k) + " outside [1, " + std::to_string(n) + "]");
    if (qdim != d) fail(ADG_EINVAL, "knn_query: query dimension mismatch");
    const std::vector<Cand> h = knn_host(ctx, database, dtype, n, d, queries, qdtype, nq, k, false);
    std::map<int, uint64_t> counts;
    for (const Cand& c : h) ++counts[labels[c.idx]];
    uint64_t best = 0;
    for (const auto& kv : counts) best = std::max(best, kv.second);
    std::vector<int> tied;
    for (const auto& kv : counts)
      if (kv.second == best) tied.push_back(kv.first);
    if (tied.size() == 1) {
      *label_out = tied.front();
      return;
    }
    HostRng rng{tie_seed};
    *label_out = tied[(size_t)rng.below(tied.size())];
  });
}

// proj/src/downstream.cpp:90-137 (build_knn_graph): symmetrised union, edges
// in (u, v) order, binary or Gaussian weights exp(-dist^2 / sigma^2) with
// sigma the median of the n k neighbour distances.
adg_status adg_build_knn_graph(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                               int k, int32_t weighting, adg_knn_edge* edges_out,
                               int64_t edges_capacity, int64_t* edges_written) {
  return guard_call([&] {
    ADG_REQUIRE(ctx && edges_written, "build_knn_graph: null argument");
    ADG_CUDA(cudaSetDevice(ctx->device));
    if (k < 1 || k >= n)
      fail(ADG_EINVAL, "build_knn_graph: k = " + std::to_string(k) + " outside [1, n)");
    ADG_REQUIRE(weighting == ADG_EDGES_BINARY || weighting == ADG_EDGES_GAUSSIAN,
                "build_knn_graph: unknown weighting");
    KnnStageTimer tm(ctx);
    cudaStream_t st = ctx->stream;
    const int64_t N = n * k;
    DevBuf<unsigned long long> keys((size_t)N, st), ukeys((size_t)N, st);
    DevBuf<double> dists((size_t)N, st), udist((size_t)N, st);
    {
      In xx(X, (size_t)(n * d) * dtype_size(dtype), st);
      DevBuf<Cand> lists((size_t)N, st);
      ctx->last_knn_engine = 2;
      if (!knn_graph_tc(ctx, xx.dev, dtype, n, d, k, lists.ptr)) {
        ctx->last_knn_engine = 1;
        knn_device(ctx, xx.dev, dtype, n, d, xx.dev, dtype, n, k, true, lists.ptr);
      }
      tm.mark("lists");
      edge_keys_kernel<<<blocks_for(N, 256), 256, 0, st>>>(lists.ptr, n, k, keys.ptr, dists.ptr);
      after_launch(ctx);
    }
    tm.mark("keys");
    // sigma = the median of the n k neighbour distances (nth_element at size/2
    // in the reference = the sorted array's element size/2)
    double sigma = 0.0;
    int bits = 1;
    while ((1LL << bits) < n) ++bits;
    DevBuf<unsigned long long> skeys((size_t)N, st);
    {
      DevBuf<double> sd((size_t)N, st);
      size_t tb = 0, tb2 = 0;
      ADG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.ptr, skeys.ptr, dists.ptr, udist.ptr,
                                               (int)N, 0, 32 + bits, st));
      if (weighting == ADG_EDGES_GAUSSIAN)
        ADG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb2, dists.ptr, sd.ptr, (int)N, 0, 64, st));
      DevBuf<uint8_t> tmp(std::max(tb, tb2), st);
      if (weighting == ADG_EDGES_GAUSSIAN) {
        ADG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.ptr, tb2, dists.ptr, sd.ptr, (int)N, 0, 64, st));
        ADG_CUDA(cudaMemcpyAsync(&sigma, sd.ptr + N / 2, sizeof(double), cudaMemcpyDeviceToHost, st));
      }
      // edge (min, max): both directions carry the same distance bits, so the
      // first insertion's weight (std::map::emplace) is any copy's weight
      ADG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, keys.ptr, skeys.ptr, dists.ptr, udist.ptr,
                                               (int)N, 0, 32 + bits, st));
    }
    DevBuf<int64_t> nsel(1, st);
    size_t tb3 = 0;
    ADG_CUDA(cub::DeviceSelect::UniqueByKey(nullptr, tb3, skeys.ptr, udist.ptr, ukeys.ptr, dists.ptr,
                                            nsel.ptr, N, st));
    DevBuf<uint8_t> tmp3(tb3, st);
    ADG_CUDA(cub::DeviceSelect::UniqueByKey(tmp3.ptr, tb3, skeys.ptr, udist.ptr, ukeys.ptr, dists.ptr,
                                            nsel.ptr, N, st));
    int64_t m = 0;
    ADG_CUDA(cudaMemcpyAsync(&m, nsel.ptr, sizeof(m), cudaMemcpyDeviceToHost, st));
    ADG_CUDA(cudaStreamSynchronize(st));
    tm.mark("sort");
    *edges_written = m;
    ADG_REQUIRE(m <= edges_capacity && (m == 0 || edges_out), "build_knn_graph: edges_out too small");
    auto* hk = static_cast<unsigned long long*>(pinned_stage(ctx, (size_t)std::max<int64_t>(m, 1) * 16));
    double* hd = reinterpret_cast<double*>(hk + m);
    ADG_CUDA(cudaMemcpyAsync(hk, ukeys.ptr, sizeof(unsigned long long) * (size_t)m, cudaMemcpyDeviceToHost, st));
    ADG_CUDA(cudaMemcpyAsync(hd, dists.ptr, sizeof(double) * (size_t)m, cudaMemcpyDeviceToHost, st));
    ADG_CUDA(cudaStreamSynchronize(st));
    tm.mark("d2h");
    // weights with the host's std::exp, as the reference (threads over slices)
    const bool gauss = weighting == ADG_EDGES_GAUSSIAN && sigma > 0.0;
    auto fill = [&](int64_t t0, int64_t t1) {
      for (int64_t t = t0; t < t1; ++t) {
        const double dd = hd[t];
        edges_out[t] = adg_knn_edge{(int32_t)(hk[t] >> 32), (int32_t)(hk[t] & 0xffffffffu),
                                    gauss ? std::exp(-dd * dd / (sigma * sigma)) : 1.0};
      }
    };
    const int nt = (int)std::min<int64_t>(8, std::max<int64_t>(1, m / 65536));
    std::vector<std::thread> pool;
    for (int i = 1; i < nt; ++i) pool.emplace_back(fill, m * i / nt, m * (i + 1) / nt);
    fill(0, m / nt);
    for (auto& th : pool) th.join();
    tm.mark("assemble");
  });
}

}  // extern "C"
