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

// Ordered Neumaier sum of v[0..count): thread k sums a fixed contiguous
// chunk, thread 0 merges the chunks in order -> bit-identical for any
// partitioning of the producers (every slot written by exactly one rank).
__global__ void ordered_sum_kernel(const double* __restrict__ v, int64_t count,
                                   double* __restrict__ out) {
  __shared__ double ps[1024], pc[1024];
  const int64_t per = (count + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per;
  int64_t e = b + per;
  if (e > count) e = count;
  double s = 0.0, c = 0.0;
  for (int64_t k = b; k < e; ++k) neu_add(s, c, v[k]);
  ps[threadIdx.x] = s;
  pc[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0.0, tc = 0.0;
    for (unsigned t = 0; t < blockDim.x; ++t) neu_add(ts, tc, ps[t] + pc[t]);
    *out = ts + tc;
  }
}

void ordered_sum(adg_ctx* ctx, const double* v, int64_t count, double* out_dev) {
  ordered_sum_kernel<<<1, 1024, 0, ctx->stream>>>(v, count, out_dev);
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
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = arg;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.0f;
    int64_t a = -1;
    for (unsigned t = 0; t < blockDim.x; ++t)
      if (bi[t] >= 0 && (bv[t] > m || (bv[t] == m && (a < 0 || bi[t] < a)))) {
        m = bv[t];
        a = bi[t];
      }
    *out = a;
  }
}

void argmax_f32(adg_ctx* ctx, const float* v, int64_t n, int64_t* out_dev) {
  argmax_f32_kernel<<<1, 1024, 0, ctx->stream>>>(v, n, out_dev);
  after_launch(ctx);
}

// Rows whose screened upper bound reaches the exact lower bound L.
__global__ void select_rows_kernel(const float* __restrict__ bound, int64_t n, float L,
                                   int64_t* __restrict__ rows, unsigned long long* __restrict__ count,
                                   int64_t cap) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (bound[k] >= L) {
      const unsigned long long s = atomicAdd(count, 1ull);
      if ((int64_t)s < cap) rows[s] = k;
    }
  }
}

void select_rows(adg_ctx* ctx, const float* bound, int64_t n, float L, int64_t* rows_dev,
                 unsigned long long* count_dev, int64_t cap) {
  select_rows_kernel<<<blocks_for(n, 256, 4 * ctx->num_sms), 256, 0, ctx->stream>>>(
      bound, n, L, rows_dev, count_dev, cap);
  after_launch(ctx);
}

}  // namespace adg
