// adg_embed.cuh -- interfaces of adg_embed.cu
#pragma once
#include "adg_internal.cuh"

#include <cmath>
#include <type_traits>

namespace adg {

void column_means(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d, double* mean);
void column_means_sampled(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d,
                          int64_t max_rows, double* mean);
void center_into(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d,
                 const double* mean, void* out);
void sample_jl_device(adg_ctx* ctx, int64_t k, int64_t d, uint64_t seed, double* out);
void normal_device(adg_ctx* ctx, uint64_t seed, int64_t count, double* out);

// Fused transform: holds W = [P ; S (I - P^T P)] (r x d) in the compute type.
struct TransformPlan {
  adg_ctx* ctx;
  int64_t s, k, d;
  bool use_f64;
  DevBuf<double> mean;
  DevBuf<double> w64;
  DevBuf<float> w32;
  DevBuf<float> meanf;
  // tensor-core path (fp32 input): W split into tf32 hi / lo planes, npad x kpad
  DevBuf<float> wh, wl, meanpad;
  int npad = 0;
  int64_t kpad = 0;
  TransformPlan(adg_ctx* c, const double* mean_dev, const double* P_dev, int64_t s,
                const double* S_dev, int64_t k, int64_t d, bool fp64);
  void run(const void* X, adg_dtype dt, int64_t n, void* Y, adg_dtype out_dt);
};

}  // namespace adg
