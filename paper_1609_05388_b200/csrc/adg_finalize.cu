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
  if (threadIdx.x != 0) return;
  double s = 0.0, c = 0.0;
  for (int t = 0; t < OS_PARTS; ++t) neu_add(s, c, parts[t]);
  *out = s + c;
}

void ordered_sum(adg_ctx* ctx, const double* v, int64_t count, double* out_dev) {
  DevBuf<double> parts(OS_PARTS, ctx->stream);
  ordered_sum_part_kernel<<<OS_PARTS, OS_THREADS, 0, ctx->stream>>>(v, count, parts.ptr);
  after_launch(ctx);
  ordered_sum_final_kernel<<<1, 32, 0, ctx->stream>>>(parts.ptr, out_dev);
  after_launch(ctx);
}

// L = exact max over the RowBest entries of one refined row (device side, so
// the candidate selection needs no host round trip).
__global__ void row_lower_bound_kernel(const double* __restrict__ best, int64_t count, int64_t stride,
                                       float* __restrict__ Lf, double* __restrict__ L) {
  if (threadIdx.x != 0) return;
  double m = -1.0;
  for (int64_t k = 0; k < count; ++k) m = fmax(m, best[k * stride]);
  *L = m;
  // float(L) rounded down a little so fp32 rounding of the bounds never drops a row
  *Lf = m >= 0.0 ? (float)(m * (1.0 - 1e-6)) : 3.0e38f;
}

void row_lower_bound(adg_ctx* ctx, const double* best, int64_t count, int64_t stride, float* Lf,
                     double* L) {
  row_lower_bound_kernel<<<1, 32, 0, ctx->stream>>>(best, count, stride, Lf, L);
  after_launch(ctx);
}

// Index of the largest non-negative float (lowest index on ties); -1 if all 0.
__global__ void argmax_f32_kernel(const float* __restrict__ v, int64_t n, int64_t* __restrict__ out) {
  __shared__ float bv[1024];
  __shared__ int64_t bi[1024];
  float best = 0.0f;
  int64_t arg = -1;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x)
    if (v[k] > best) {
      best = v[k];
      arg = k;
    }
  // warp then block reduction: larger value wins, lower index on ties
  auto better = [](float v1, int64_t i1, float v2, int64_t i2) {
    if (i2 < 0) return false;
    if (i1 < 0) return true;
    return v2 > v1 || (v2 == v1 && i2 < i1);
  };
  for (int s = 16; s; s >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, s);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, arg, s);
    if (better(best, arg, ov, oi)) {
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
    float m = 0.0f;
    int64_t a = -1;
    for (unsigned w = 0; w < blockDim.x / 32; ++w)
      if (better(m, a, bv[w], bi[w])) {
        m = bv[w];
        a = bi[w];
      }
    *out = a;
  }
}

void argmax_f32(adg_ctx* ctx, const float* v, int64_t n, int64_t* out_dev) {
  argmax_f32_kernel<<<1, 1024, 0, ctx->stream>>>(v, n, out_dev);
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
