// adg_eval.cuh -- device-resident evaluation entry points shared by the C ABI
// (adg_api.cu) and the sweep module (adg_sweep.cu).
#pragma once
#include "adg_internal.cuh"

namespace adg {

// proj/src/distortion.cpp:113-192 on device clouds (arguments already
// validated); report / hist_out (hist_bins + 1) are host memory.
void evaluate_device(adg_ctx* ctx, const void* xdev, adg_dtype orig_dtype, int64_t n, int64_t d,
                     const void* ydev, adg_dtype emb_dtype, int64_t r, const adg_pair_sampling* mode,
                     int hist_bins, double hist_max, adg_engine engine, adg_report* report,
                     uint64_t* hist_out);

// proj/src/distortion.cpp:194-196 (evaluate(all).max_distortion) -- or the
// max of the given sampling mode -- on device clouds.  All-pairs jobs beyond
// the exact engine's range use the SCREEN engine in max-only mode (no
// histogram, no sums); the value is the reference's exactly (fp64 refine).
// upper != nullptr: bounds only -- the return value L (the exact maximum of
// the row holding the screened maximum, and of the near-coincident pairs) and
// *upper U bracket the exact maximum, L <= max <= U, without the exact refine
// of the other candidate rows; U == L when that refine would be empty.
double max_distortion_device(adg_ctx* ctx, const void* xdev, adg_dtype xd, int64_t n, int64_t d,
                             const void* ydev, adg_dtype yd, int64_t r,
                             const adg_pair_sampling* mode, double* upper = nullptr);

}  // namespace adg
