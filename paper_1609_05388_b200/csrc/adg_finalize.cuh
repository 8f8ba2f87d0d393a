// adg_finalize.cuh -- interfaces of adg_finalize.cu
#pragma once
#include "adg_internal.cuh"

namespace adg {
void ordered_sum(adg_ctx* ctx, const double* v, int64_t count, double* out_dev);
void argmax_f32(adg_ctx* ctx, const float* v, int64_t n, int64_t* out_dev);
void select_rows(adg_ctx* ctx, const float* bound, int64_t n, float L, int64_t* rows_dev,
                 unsigned long long* count_dev, int64_t cap);
}  // namespace adg
