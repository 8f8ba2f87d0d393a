// adg_exact.cuh -- interfaces of adg_exact.cu
#pragma once
#include "adg_internal.cuh"

namespace adg {

struct BlockOut {
  double sum;  // Neumaier total of the block
  double max;  // -1 when nothing evaluated
  uint64_t argp;
  uint64_t evaluated;
  uint64_t zero;
};

struct MergeOut {
  double sum;
  double max;
  uint64_t argp;
  uint64_t evaluated;
  uint64_t zero;
};

struct RowBest {
  double max;  // -1 when the row had no evaluated pair
  int64_t i;
  int64_t j;
};

// All pairs (sampled == nullptr, work = n(n-1)/2) or the listed linear pair
// indices (sampled[work], sorted).  hist_dev (bins+1) is accumulated into.
void run_exact(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d, const void* Y,
               adg_dtype yd, int64_t r, const uint64_t* sampled, uint64_t work, int bins,
               double hist_max, unsigned long long* hist_dev, MergeOut* merged_dev);

// All pairs of large clouds (n > 4096): the same per-pair values, counts,
// histogram, max and argmax as run_exact, staged through 64 x 64 shared-memory
// pair tiles (adg_exact_tiled.cu); the mean's summation order is per tile.
void run_exact_tiled(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d, const void* Y,
                     adg_dtype yd, int64_t r, int bins, double hist_max,
                     unsigned long long* hist_dev, MergeOut* merged_dev);

int64_t row_refine_chunks(int64_t n);  // RowBest entries per refined row
// One row's chunks [chunk0, chunk1) of the single-row refine (out_dev gets
// chunk1 - chunk0 entries): a rank's share in the sharded evaluator.
void run_row_refine_chunks(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d,
                           const void* Y, adg_dtype yd, int64_t r, const int64_t* row_dev,
                           int64_t chunk0, int64_t chunk1, RowBest* out_dev);
void run_row_refine(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d, const void* Y,
                    adg_dtype yd, int64_t r, const int64_t* rows_dev, int64_t nrows,
                    RowBest* out_dev, int64_t* chunks_per_row_out);

void run_pair_list(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t d, const void* Y,
                   adg_dtype yd, int64_t r, const uint32_t* pairs_dev, int64_t count,
                   double* values_dev);

// Exact binning of the SCREEN's edge list (entries [0, min(*count, cap)),
// sentinel slots skipped), added into hist_dev (bins + 1); *binned_dev counts
// them.  When the list
// overflowed (*count > cap), *near_count_dev is raised to near_cap + 1 (if
// given): the finalize then redoes the histogram in tile chunks.
void run_edge_bin(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t d, const void* Y,
                  adg_dtype yd, int64_t r, const uint2* pairs_dev,
                  const unsigned long long* count_dev, int64_t cap, int bins, double hist_max,
                  unsigned long long* hist_dev, unsigned long long* binned_dev,
                  unsigned long long* near_count_dev = nullptr, int64_t near_cap = 0);

}  // namespace adg
