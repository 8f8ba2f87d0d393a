// adg_finalize.cu -- small deterministic reductions used after the screen.
#include "adg_finalize.cuh"

namespace adg {

__device__ __forceinline__ void neu_add(double& s, double& c, double v) {
  const double t = s + v;
  if (fabs(s) >= fabs(v))
    c += (s - t) + v;
  else
    c += (v - t) + s;
  s = t;
}

// Ordered Neumaier sum of v[0..count) in two fixed levels: OS_PARTS chunks
// (a function of count only, never of the GPU), each summed by one CTA whose
// threads own fixed sub-chunks merged in thread order, then the chunk totals
// merged in order -> bit-identical for any partitioning of the producers
// (every slot written by exactly one rank) and any device.
constexpr int OS_PARTS = 256, OS_THREADS = 256;

__global__ void ordered_sum_part_kernel(const double* __restrict__ v, int64_t count,
                                        double* __restrict__ parts) {
  __shared__ double ps[OS_THREADS];
  const int64_t per_part = (count + OS_PARTS - 1) / OS_PARTS;
  const int64_t p0 = (int64_t)blockIdx.x * per_part;
  int64_t p1 = p0 + per_part;
  if (p1 > count) p1 = count;
  const int64_t per = (per_part + OS_THREADS - 1) / OS_THREADS;
  const int64_t b = p0 + threadIdx.x * per;
  int64_t e = b + per;
  if (e > p1) e = p1;
  double s = 0.0, c = 0.0;
  for (int64_t k = b; k < e; ++k) neu_add(s, c, v[k]);
  ps[threadIdx.x] = s + c;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0.0, tc = 0.0;
    for (int t = 0; t < OS_THREADS; ++t) neu_add(ts, tc, ps[t]);
    parts[blockIdx.x] = ts + tc;
  }
}

__global__ void ordered_sum_final_kernel(const double* __restrict__ parts, double* __restrict__ out) {
  // stage the chunk totals with one coalesced load each, then merge them in
  // order from shared memory (the same sequence of Neumaier additions)
  __shared__ double ps[OS_PARTS];
  for (int t = threadIdx.x; t < OS_PARTS; t += blockDim.x) ps[t] = parts[t];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double s = 0.0, c = 0.0;
  for (int t = 0; t < OS_PARTS; ++t) neu_add(s, c, ps[t]);
  *out = s + c;
}

void ordered_sum(adg_ctx* ctx, const double* v, int64_t count, double* out_dev) {
  DevBuf<double> parts(OS_PARTS, ctx->stream);
  ordered_sum_part_kernel<<<OS_PARTS, OS_THREADS, 0, ctx->stream>>>(v, count, parts.ptr);
  after_launch(ctx);
  ordered_sum_final_kernel<<<1, OS_THREADS, 0, ctx->stream>>>(parts.ptr, out_dev);
  after_launch(ctx);
}

// L = exact max over the RowBest entries of one refined row (device side, so
// the candidate selection needs no host round trip).
__global__ void row_lower_bound_kernel(const double* __restrict__ best, int64_t count, int64_t stride,
                                       float* __restrict__ Lf, double* __restrict__ L) {
  // max is exact in any order: strided loads over the block, then a tree
  __shared__ double wm[32];
  double m = -1.0;
  for (int64_t k = threadIdx.x; k < count; k += blockDim.x) m = fmax(m, best[k * stride]);
  for (int s = 16; s; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (unsigned w = 1; w < blockDim.x / 32; ++w) m = fmax(m, wm[w]);
  *L = m;
  // float(L) rounded down a little so fp32 rounding of the bounds never drops a row
  *Lf = m >= 0.0 ? (float)(m * (1.0 - 1e-6)) : 3.0e38f;
}

void row_lower_bound(adg_ctx* ctx, const double* best, int64_t count, int64_t stride, float* Lf,
                     double* L) {
  row_lower_bound_kernel<<<1, 256, 0, ctx->stream>>>(best, count, stride, Lf, L);
  after_launch(ctx);
}

// Index of the largest non-negative float (lowest index on ties); -1 if all 0.
// Two levels: AM_PARTS CTAs each take a contiguous chunk (16-byte loads), then
// one CTA merges the chunk winners in chunk order.
constexpr int AM_PARTS = 128, AM_THREADS = 256;

struct ArgBest {
  float v;
  int64_t i;
};

__device__ __forceinline__ bool am_better(float v1, int64_t i1, float v2, int64_t i2) {
  if (i2 < 0) return false;
  if (i1 < 0) return true;
  return v2 > v1 || (v2 == v1 && i2 < i1);
}

__device__ __forceinline__ void am_block_reduce(float& best, int64_t& arg) {
  __shared__ float bv[32];
  __shared__ int64_t bi[32];
  for (int s = 16; s; s >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, s);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, arg, s);
    if (am_better(best, arg, ov, oi)) {
      best = ov;
      arg = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = best;
    bi[threadIdx.x >> 5] = arg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (unsigned w = 1; w < blockDim.x / 32; ++w)
      if (am_better(best, arg, bv[w], bi[w])) {
        best = bv[w];
        arg = bi[w];
      }
  }
}

__global__ void __launch_bounds__(AM_THREADS) argmax_part_kernel(const float* __restrict__ v, int64_t n,
                                                                 ArgBest* __restrict__ parts) {
  const int64_t per = ((n + AM_PARTS - 1) / AM_PARTS + 3) / 4 * 4;  // multiple of 4: aligned float4 chunks
  const int64_t b = (int64_t)blockIdx.x * per;
  int64_t e = b + per;
  if (e > n) e = n;
  float best = 0.0f;
  int64_t arg = -1;
  const bool vec = (reinterpret_cast<uintptr_t>(v) & 15) == 0;
  if (vec) {
    for (int64_t k = b + 4 * threadIdx.x; k < e; k += 4 * AM_THREADS) {
      if (k + 3 < e) {
        const float4 q = *reinterpret_cast<const float4*>(v + k);
        if (q.x > best) best = q.x, arg = k;
        if (q.y > best) best = q.y, arg = k + 1;
        if (q.z > best) best = q.z, arg = k + 2;
        if (q.w > best) best = q.w, arg = k + 3;
      } else {
        for (int64_t t = k; t < e; ++t)
          if (v[t] > best) best = v[t], arg = t;
      }
    }
  } else {
    for (int64_t k = b + threadIdx.x; k < e; k += AM_THREADS)
      if (v[k] > best) best = v[k], arg = k;
  }
  am_block_reduce(best, arg);
  if (threadIdx.x == 0) parts[blockIdx.x] = ArgBest{best, arg};
}

__global__ void argmax_final_kernel(const ArgBest* __restrict__ parts, int64_t* __restrict__ out) {
  float best = 0.0f;
  int64_t arg = -1;
  for (int t = threadIdx.x; t < AM_PARTS; t += blockDim.x)
    if (am_better(best, arg, parts[t].v, parts[t].i)) {
      best = parts[t].v;
      arg = parts[t].i;
    }
  am_block_reduce(best, arg);
  if (threadIdx.x == 0) *out = arg;
}

void argmax_f32(adg_ctx* ctx, const float* v, int64_t n, int64_t* out_dev) {
  DevBuf<ArgBest> parts(AM_PARTS, ctx->stream);
  argmax_part_kernel<<<AM_PARTS, AM_THREADS, 0, ctx->stream>>>(v, n, parts.ptr);
  after_launch(ctx);
  argmax_final_kernel<<<1, AM_PARTS, 0, ctx->stream>>>(parts.ptr, out_dev);
  after_launch(ctx);
}

// Rows whose screened upper bound reaches the exact lower bound L.
__global__ void select_rows_kernel(const float* __restrict__ bound, int64_t n, const float* __restrict__ Lp,
                                   int64_t* __restrict__ rows, unsigned long long* __restrict__ count,
                                   int64_t cap) {
  const float L = *Lp;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (bound[k] >= L) {
      const unsigned long long s = atomicAdd(count, 1ull);
      if ((int64_t)s < cap) rows[s] = k;
    }
  }
}

void select_rows(adg_ctx* ctx, const float* bound, int64_t n, const float* L_dev, int64_t* rows_dev,
                 unsigned long long* count_dev, int64_t cap) {
  select_rows_kernel<<<blocks_for(n, 256, 4 * ctx->num_sms), 256, 0, ctx->stream>>>(
      bound, n, L_dev, rows_dev, count_dev, cap);
  after_launch(ctx);
}

}  // namespace adg
