// adg_screen.cuh -- interfaces of adg_screen.cu
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include <map>
#include <vector>

#include "adg_embed.cuh"

namespace adg {

using TileListCache = std::map<int64_t, DevBuf<uint32_t>>;  // adg_ctx::tile_lists
void free_tile_list_cache(adg_ctx* ctx);

// Device operands of the SCREEN engine (built once per evaluation plan).
// The screen's centring shift (conditioning only; distances are
// shift-invariant): mean of <= kShiftRows evenly spaced rows, zeroed for bf16 rows
// that are nearly centred already so their fp16 planes stay exact.
void screen_shift(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d, double* mx);
// rows sampled (evenly spaced) for the centring shifts (conditioning only)
// -- the pipelined run_distort flow copies them from the host with one
// strided copy ahead of the first row chunk
constexpr int64_t kShiftRows = 1024;

struct ScreenOperands {
  adg_ctx* ctx;
  int64_t n, d, r;
  int64_t T = 0, rows_pad = 0, kp = 0, kr = 0, ktot = 0;
  DevBuf<__half> hi, lo;
  DevBuf<float4> meta;
  DevBuf<int> lo_flag;  // set by the prep when any original-side lo entry is non-zero
  const uint32_t* tiles_ptr = nullptr;  // the list in use (banded or phased: cached per context)
  const uint32_t* slots_ptr = nullptr;  // canonical slot per listed tile
  // the banded list as tile pairs sharing their 256-row block (screen_mc_kernel:
  // entry 2 k + pair, 0xFFFFFFFF = no tile), with slots; cached per context
  const uint32_t* mc_tiles_ptr = nullptr;
  const uint32_t* mc_slots_ptr = nullptr;
  int64_t mc_pairs = 0;
  int64_t num_tiles = 0;
  CUtensorMap map_a_hi, map_a_lo, map_b_hi, map_b_lo;  // 128-row (A) / 64-row (B) boxes
  float eps = 0.f, tau = 0.f;
  int kc_orig = 0, kc_total = 0, k16_last_orig = 0, k16_last_emb = 0;
  std::vector<int64_t> phase_tile_end;  // phased lists: phase k = tiles [end[k-1], end[k])
  // centre (sampled-row means), prep every row, banded tile list
  ScreenOperands(adg_ctx* c, const void* X, adg_dtype xd, int64_t n, int64_t d, const void* Y,
                 adg_dtype yd, int64_t r);
  // planes, maps and tile list only (phased by phase_rows if given); rows are
  // prepared later with prep_rows, e.g. as they arrive from the host
  ScreenOperands(adg_ctx* c, int64_t n, int64_t d, int64_t r, const std::vector<int64_t>* phase_rows);
  void prep_rows(const void* X, adg_dtype xd, const void* Y, adg_dtype yd, const double* mx,
                 const double* my, int64_t row0, int64_t row1);
  // re-read X / Y (same shapes): centring shift, exact-plane flag, every row
  void refresh(const void* X, adg_dtype xd, const void* Y, adg_dtype yd);

 private:
  void setup(const std::vector<int64_t>* phase_rows);
};

struct ScreenPartials {
  unsigned long long* hist;
  double* tile_sums;
  float* row_max;
  float* row_bound;
  uint32_t* near_pairs;
  unsigned long long* near_count;
  long long near_cap;
  uint2* edge_pairs;  // pairs too close to a bin edge (exact re-binning)
  unsigned long long* edge_count;
  long long edge_cap;
  float edge_f;  // edge band in units of the per-pair error bound (0: none)
};

std::vector<uint32_t> build_tile_list(int64_t n, int64_t band);
// rows blocks per band of the tile list for planes of ktot columns
int64_t screen_band(int64_t ktot);
std::vector<uint32_t> tile_slots(const std::vector<uint32_t>& tiles, int64_t n);
struct ScreenConfig {
  int stages;
  int hmode;  // histogram mode of screen_kernel (adg_screen_kernel.cuh)
  size_t smem;
  bool global_hist = false;  // HMODE 0 counters in per-CTA global scratch
};
// Edge band of the exact-histogram mode, as a fraction of the rigorous
// per-pair bound.  The worst screened error measured on C3 (all 1.8e9 pairs)
// lies between 1/16 and 1/8 of the bound (fp32 accumulation in the tensor
// core drifts systematically), so 1/4 keeps a 2x margin
// (profiles/r02_edge_band.md).
constexpr double kScreenEdgeBand = 0.25;
double screen_edge_band(bool exact_hist);
ScreenConfig screen_config(int bins);
int screen_tile_slots();  // tile_sums slots per tile (one per epilogue warp)
// max_only: per-row max / bound and the near-coincident list only (no
// histogram, no sums) -- for max_distortion and the sweep probes.
// stream: the context's (default) or another one (e.g. the pipelined flow's
// phases, which run concurrently: their partial updates are order-free)
void run_screen(adg_ctx* ctx, const ScreenOperands& ops, int64_t tile_begin, int64_t tile_end,
                int bins, double hist_max, const ScreenPartials& out, bool max_only = false,
                cudaStream_t stream = nullptr);
// HMODE 4: append {query, candidate, lo, hi} for every pair within either
// side's radius sqrt(tau2) (ops with r = 0); *count = slots used (may exceed cap)
void run_screen_knn(adg_ctx* ctx, const ScreenOperands& ops, const float* tau2, uint4* out,
                    unsigned long long* count, long long cap);

}  // namespace adg
