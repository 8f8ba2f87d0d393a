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
#include <cmath>
#include <map>
#include <vector>

#include "adg_internal.cuh"

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

std::vector<Cand> knn_host(adg_ctx* ctx, const void* D, adg_dtype dd, int64_t n, int64_t d,
                           const void* Q, adg_dtype qd, int64_t nq, int k, bool skip_self) {
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
    const std::vector<Cand> h = knn_host(ctx, X, dtype, n, d, X, dtype, n, k, true);
    double sigma = 0.0;
    if (weighting == ADG_EDGES_GAUSSIAN) {
      std::vector<double> dist(h.size());
      for (size_t t = 0; t < h.size(); ++t) dist[t] = h[t].dist;
      std::nth_element(dist.begin(), dist.begin() + dist.size() / 2, dist.end());
      sigma = dist[dist.size() / 2];
    }
    // edge (min, max) with the weight of its first insertion in u order
    // (std::map::emplace keeps the first; both directions give the same dist)
    std::vector<std::pair<std::pair<int, int>, double>> e;
    e.reserve(h.size());
    for (int64_t u = 0; u < n; ++u)
      for (int b = 0; b < k; ++b) {
        const Cand& c = h[(size_t)(u * k + b)];
        const int a = (int)std::min<int64_t>(u, c.idx), bb = (int)std::max<int64_t>(u, c.idx);
        double w = 1.0;
        if (weighting == ADG_EDGES_GAUSSIAN && sigma > 0.0) w = std::exp(-c.dist * c.dist / (sigma * sigma));
        e.push_back({{a, bb}, w});
      }
    std::stable_sort(e.begin(), e.end(),
                     [](const auto& x, const auto& y) { return x.first < y.first; });
    int64_t m = 0;
    for (size_t t = 0; t < e.size(); ++t) {
      if (t > 0 && e[t].first == e[t - 1].first) continue;
      if (m < edges_capacity && edges_out)
        edges_out[m] = adg_knn_edge{e[t].first.first, e[t].first.second, e[t].second};
      ++m;
    }
    *edges_written = m;
    ADG_REQUIRE(m <= edges_capacity, "build_knn_graph: edges_out too small");
  });
}

}  // extern "C"
