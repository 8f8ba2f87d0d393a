// adg_finalize.cuh -- interfaces of adg_finalize.cu
#pragma once
#include "adg_internal.cuh"

namespace adg {
void ordered_sum(adg_ctx* ctx, const double* v, int64_t count, double* out_dev);
void argmax_f32(adg_ctx* ctx, const float* v, int64_t n, int64_t* out_dev);
// best: RowBest array viewed as doubles (max at stride 0, entry stride in doubles)
void row_lower_bound(adg_ctx* ctx, const double* best, int64_t count, int64_t stride, float* Lf,
                     double* L);
void select_rows(adg_ctx* ctx, const float* bound, int64_t n, const float* L_dev, int64_t* rows_dev,
                 unsigned long long* count_dev, int64_t cap);
}  // namespace adg
