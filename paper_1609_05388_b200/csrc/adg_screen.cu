// adg_screen.cu -- SCREEN engine of the all-pairs distortion evaluator.
//
// Replaces the O(n^2 (d+r)) loop of proj/src/distortion.cpp:139-169 for large
// jobs.  Pairwise squared distances are formed in Gram form on the 5th-gen
// tensor cores:  o_ij = |x_i|^2 + |x_j|^2 - 2 x_i.x_j  (and e_ij likewise for
// the embedded points), with the dot products from tcgen05.mma (kind::f16,
// fp32 accumulation in TMEM) over a split-fp16 representation of the centred
// rows: x~ * 2^e_i = hi + lo (both fp16, per-row power-of-two scale so the
// row max lands in [2^14, 2^15)), and x.y ~ hi.hi + hi.lo + lo.hi (3 MMAs per
// K step).  That keeps ~22 mantissa bits through the |x|^2+|y|^2-2x.y
// cancellation.  The epilogue forms |sqrt(e/o) - 1| in registers and reduces,
// per pair and without materialising anything n x n:
//   * the histogram (distortion.cpp:81-87 binning) in per-thread u8 smem
//     counters, flushed to a per-CTA u32 histogram and then to global u64,
//   * per-tile partial sums (deterministic slots, ordered reduction later),
//   * per-row screened max and screened max + rigorous error bound, which the
//     exact fp64 refine (adg_exact.cu) uses to recover the reference's max
//     and its lowest (i, j) argmax exactly,
//   * pairs whose screened o is within the noise of 0 (possible duplicates),
//     listed for the exact zero rule of distortion.cpp:66-69.
// The kernel itself (2-CTA tcgen05 pipeline) is in adg_screen_kernel.cuh.
#include "adg_screen.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>

#include "adg_finalize.cuh"
#include "adg_prep.cuh"
#include "adg_screen_kernel.cuh"
#include "adg_tma.cuh"

namespace adg {

// ------------------------------------------------------------ prep kernel
// One warp per padded row: centre (fp64), pick the power-of-two scale, write
// the hi/lo fp16 planes ([rows_pad][ktot], orig at [0,d), emb at [kp, kp+r)),
// and the row metadata computed from the represented value hi+lo.
template <typename TO, typename TE>
__global__ void prep_kernel(const TO* __restrict__ X, int64_t n, int64_t d,
                            const double* __restrict__ mx, const TE* __restrict__ Y, int64_t r,
                            const double* __restrict__ my, int64_t rows_pad, int64_t kp,
                            int64_t ktot, __half* __restrict__ hi, __half* __restrict__ lo,
                            float4* __restrict__ meta, int64_t row0, int64_t row1, int* lo_flag) {
  const int64_t row = row0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= row1 || row >= rows_pad) return;
  __half* hrow = hi + row * ktot;
  __half* lrow = lo + row * ktot;
  if (row >= n) {
    for (int64_t t = lane; t < ktot; t += 32) {
      hrow[t] = __float2half(0.0f);
      lrow[t] = __float2half(0.0f);
    }
    if (lane == 0) meta[row] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  float4 m4;
  bool lnz = false;
  for (int part = 0; part < 2; ++part) {
    const int64_t len = part == 0 ? d : r;
    const int64_t off = part == 0 ? 0 : kp;
    const int64_t end = part == 0 ? kp : ktot;
    double amax = 0.0;
    for (int64_t t = lane; t < len; t += 32) {
      const double v = part == 0 ? to_f64(X[row * d + t]) - mx[t] : to_f64(Y[row * r + t]) - my[t];
      amax = fmax(amax, fabs(v));
    }
    for (int s = 16; s; s >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, s));
    int ex = 0;
    if (amax > 0.0) frexp(amax, &ex);  // amax in [2^(ex-1), 2^ex)
    const int e = amax > 0.0 ? 15 - ex : 0;
    double nrm = 0.0;
    for (int64_t t = lane; t < end - off; t += 32) {
      double v = 0.0;
      if (t < len)
        v = part == 0 ? to_f64(X[row * d + t]) - mx[t] : to_f64(Y[row * r + t]) - my[t];
      const double sv = ldexp(v, e);
      const __half h = __float2half_rn((float)sv);
      const double rest = sv - (double)__half2float(h);
      const __half l = __float2half_rn((float)rest);
      hrow[off + t] = h;
      lrow[off + t] = l;
      lnz = lnz || (part == 0 && half_nonzero(l));
      const double rep = (double)__half2float(h) + (double)__half2float(l);
      nrm = fma(rep, rep, nrm);
    }
    for (int s = 16; s; s >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, s);
    const double inv = ldexp(1.0, -e);
    if (part == 0) {
      m4.x = (float)(nrm * inv * inv);
      m4.z = (float)inv;
    } else {
      m4.y = (float)(nrm * inv * inv);
      m4.w = (float)inv;
    }
  }
  note_lo(lnz, lo_flag);
  if (lane == 0) meta[row] = m4;
}

// fp32 / bf16 inputs: the same split in fp32 arithmetic.  x - (float)mean
// rounds at 2^-24 relative (below the split's 2^-22), the rounding of the
// mean itself is a constant shift of every row (invisible to distances), and
// the power-of-two scaling and sv - hi are exact; only the norm accumulates in
// fp64.  One warp per row, two passes (max, then split), the second from L1/L2.
template <typename TO, typename TE>
__global__ void __launch_bounds__(256)
prep_f32_kernel(const TO* __restrict__ X, int64_t n, int64_t d, const double* __restrict__ mx,
                const TE* __restrict__ Y, int64_t r, const double* __restrict__ my, int64_t rows_pad,
                int64_t kp, int64_t ktot, __half* __restrict__ hi, __half* __restrict__ lo,
                float4* __restrict__ meta, int64_t row0, int64_t row1, int* lo_flag) {
  const int64_t row = row0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= row1 || row >= rows_pad) return;
  __half* hrow = hi + row * ktot;
  __half* lrow = lo + row * ktot;
  if (row >= n) {
    for (int64_t t = lane; t < ktot; t += 32) {
      hrow[t] = __float2half(0.0f);
      lrow[t] = __float2half(0.0f);
    }
    if (lane == 0) meta[row] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  float4 m4;
  bool lnz = false;
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    const int64_t len = part == 0 ? d : r;
    const int64_t off = part == 0 ? 0 : kp;
    const int64_t end = part == 0 ? kp : ktot;
    float amax = 0.0f;
    for (int64_t t = lane; t < len; t += 32) {
      const float v = part == 0 ? ld_f(X + row * d + t) - (float)mx[t]
                                : ld_f(Y + row * r + t) - (float)my[t];
      amax = fmaxf(amax, fabsf(v));
    }
    for (int s = 16; s; s >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, s));
    int ex = 0;
    if (amax > 0.0f) frexpf(amax, &ex);  // amax in [2^(ex-1), 2^ex)
    const int e = amax > 0.0f ? 15 - ex : 0;
    const float scale = ldexpf(1.0f, e);
    double nrm = 0.0;
    for (int64_t t = lane; t < end - off; t += 32) {
      float v = 0.0f;
      if (t < len)
        v = part == 0 ? ld_f(X + row * d + t) - (float)mx[t] : ld_f(Y + row * r + t) - (float)my[t];
      const float sv = v * scale;
      const __half h = __float2half_rn(sv);
      const __half l = __float2half_rn(sv - __half2float(h));
      hrow[off + t] = h;
      lrow[off + t] = l;
      lnz = lnz || (part == 0 && half_nonzero(l));
      const double rep = (double)(__half2float(h) + __half2float(l));
      nrm = fma(rep, rep, nrm);
    }
    for (int s = 16; s; s >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, s);
    const double inv = ldexp(1.0, -e);
    if (part == 0) {
      m4.x = (float)(nrm * inv * inv);
      m4.z = (float)inv;
    } else {
      m4.y = (float)(nrm * inv * inv);
      m4.w = (float)inv;
    }
  }
  note_lo(lnz, lo_flag);
  if (lane == 0) meta[row] = m4;
}

// Vectorised variant for the original side when rows are 16/8-byte aligned
// (d % 4 == 0): one warp per row, prep_row (adg_prep.cuh) -- the same code
// the fused embed + prep kernel runs, so both write identical operands.  Same
// arithmetic as prep_f32_kernel, element by element.
template <typename TO, typename TE, int NV>
__global__ void __launch_bounds__(256)
prep_vec_kernel(const TO* __restrict__ X, int64_t n, int64_t d, const double* __restrict__ mx,
                const TE* __restrict__ Y, int64_t r, const double* __restrict__ my, int64_t rows_pad,
                int64_t kp, int64_t ktot, __half* __restrict__ hi, __half* __restrict__ lo,
                float4* __restrict__ meta, int64_t row0, int64_t row1, int* lo_flag) {
  // the centring shifts, rounded to fp32 once per CTA (as every element used
  // them) and read back as 16-byte shared loads
  extern __shared__ float4 prep_sh4[];
  float* msx = reinterpret_cast<float*>(prep_sh4);  // d (padded to 4)
  float* msy = msx + ((d + 3) & ~3LL);             // r
  for (int64_t t = threadIdx.x; t < d; t += blockDim.x) msx[t] = (float)mx[t];
  for (int64_t t = threadIdx.x; t < r; t += blockDim.x) msy[t] = (float)my[t];
  __syncthreads();
  const int64_t row = row0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= row1 || row >= rows_pad) return;
  const bool lnz = prep_row<TO, TE, NV>(row < n ? X + row * d : nullptr, Y + row * r, d, r, kp, ktot,
                                        prep_sh4, msy, hi + row * ktot, lo + row * ktot, meta + row, lane);
  if (row < n) note_lo(lnz, lo_flag);
}

// ----------------------------------------------------------- host side
static CUtensorMap make_plane_map(const __half* base, int64_t rows, int64_t ktot, int box_rows) {
  return make_tensor_map_2d(base, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, (uint64_t)ktot, (uint64_t)rows,
                            (uint64_t)(ktot * 2), SC_BK, (uint32_t)box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Pair tiles (I2, J): 256-row block I2 x 128-col block J with J >= 2*I2 (upper
// triangle), walked in bands of SC_BAND row blocks: for each band, every
// column block, then the band's row blocks -- consecutive tiles share A or B.
// The band's A rows (both planes, all ktot columns) should stay L2-resident
// while its column blocks stream: up to SC_BAND row blocks, halved while the
// band would exceed ~72 MB of the 126 MB L2 (C3 / C4: 32 blocks = 29 / 34 MB;
// C5, ktot = 4224: 16 blocks = 69 MB -- 219 -> 189 ms against 32).  A pure
// function of ktot, so every rank of a sharded run builds the same list.
int64_t screen_band(int64_t ktot) {
  const char* e = std::getenv("ADG_SCREEN_BAND");  // profiling aid; multi-GPU needs the default
  const int64_t b = e ? std::atoll(e) : 0;
  if (b > 0) return b;
  int64_t band = SC_BAND;
  const int64_t row_bytes = 2 * 2 * ktot;  // hi + lo fp16
  while (band > 4 && band * SC_PM * row_bytes > (72ll << 20)) band /= 2;
  return band;
}

// Pair tiles (I2, J): 256-row block I2 x 160-column block J, every J whose
// columns reach past the block's first row (J >= jmin(I2) = floor(256 I2 / 160),
// the upper triangle with the diagonal tiles), walked in bands of SC_BAND row
// blocks: for each band, every column block, then the band's row blocks.
// n is the number of points (T2 = ceil(n / 256) row blocks, T = ceil(n / 160)).
static inline int64_t tile_jmin(int64_t I2) { return I2 * SC_PM / SC_BN; }

std::vector<uint32_t> build_tile_list(int64_t n, int64_t band) {
  const int64_t T = (n + SC_BN - 1) / SC_BN, T2 = (n + SC_PM - 1) / SC_PM;
  std::vector<uint32_t> tiles;
  for (int64_t B0 = 0; B0 < T2; B0 += band) {
    const int64_t B1 = std::min<int64_t>(B0 + band, T2);
    for (int64_t J = tile_jmin(B0); J < T; ++J)
      for (int64_t I2 = B0; I2 < B1 && tile_jmin(I2) <= J; ++I2)
        tiles.push_back((uint32_t)((I2 << 16) | J));
  }
  return tiles;
}

// canonical slot of each tile: its index in row-major (I2, then J) order
std::vector<uint32_t> tile_slots(const std::vector<uint32_t>& tiles, int64_t n) {
  const int64_t T = (n + SC_BN - 1) / SC_BN, T2 = (n + SC_PM - 1) / SC_PM;
  std::vector<int64_t> off((size_t)T2 + 1, 0);
  for (int64_t i = 0; i < T2; ++i) off[(size_t)i + 1] = off[(size_t)i] + (T - tile_jmin(i));
  std::vector<uint32_t> slots(tiles.size());
  for (size_t t = 0; t < tiles.size(); ++t) {
    const int64_t I2 = tiles[t] >> 16, J = tiles[t] & 0xFFFF;
    slots[t] = (uint32_t)(off[(size_t)I2] + J - tile_jmin(I2));
  }
  return slots;
}

// The banded walk as tile pairs for screen_mc_kernel: within each band, the
// column blocks two at a time, and for each row block of the band the pair
// (I2, J), (I2, J + 1) -- both tiles read the same 256 rows (A), which the
// two CTA pairs of a 4-CTA cluster share by multicast.  A tile without a
// partner (the triangle's edge, an odd last column block) is paired with
// SC_DUMMY.  Every tile of build_tile_list appears exactly once.
static std::vector<uint32_t> build_tile_pairs(int64_t n, int64_t band) {
  const int64_t T = (n + SC_BN - 1) / SC_BN, T2 = (n + SC_PM - 1) / SC_PM;
  std::vector<uint32_t> out;
  for (int64_t B0 = 0; B0 < T2; B0 += band) {
    const int64_t B1 = std::min<int64_t>(B0 + band, T2);
    for (int64_t J = tile_jmin(B0); J < T; J += 2)
      for (int64_t I2 = B0; I2 < B1 && tile_jmin(I2) <= J + 1; ++I2) {
        const bool a = tile_jmin(I2) <= J, b = J + 1 < T;
        if (!a && !b) continue;
        const uint32_t ta = (uint32_t)((I2 << 16) | J), tb = (uint32_t)((I2 << 16) | (J + 1));
        if (a && b) {
          out.push_back(ta);
          out.push_back(tb);
        } else {
          out.push_back(a ? ta : tb);
          out.push_back(SC_DUMMY);
        }
      }
  }
  return out;
}

// Tiles in phases: phase k holds the tiles whose rows all lie below
// phase_rows[k] (a tile (I2, J) reads rows < max(256 (I2 + 1), 128 (J + 1))),
// each phase in band order -- for a pipeline that screens rows as they arrive.
static std::vector<uint32_t> phase_tiles(const std::vector<uint32_t>& banded,
                                         const std::vector<int64_t>& phase_rows,
                                         std::vector<int64_t>& phase_end) {
  std::vector<std::vector<uint32_t>> per((size_t)phase_rows.size());
  for (const uint32_t t : banded) {
    const int64_t I2 = t >> 16, J = t & 0xFFFF;
    const int64_t need = std::max<int64_t>((I2 + 1) * SC_PM, (J + 1) * SC_BN);
    size_t k = 0;
    while (k + 1 < phase_rows.size() && phase_rows[k] < need) ++k;
    per[k].push_back(t);
  }
  std::vector<uint32_t> out;
  phase_end.clear();
  for (const auto& v : per) {
    out.insert(out.end(), v.begin(), v.end());
    phase_end.push_back((int64_t)out.size());
  }
  return out;
}

void free_tile_list_cache(adg_ctx* ctx) {
  auto* m = static_cast<TileListCache*>(ctx->tile_lists);
  if (!m) return;
  for (auto& kv : *m) {  // pool memory: plain cudaFree (the allocating stream may be gone)
    cudaFree(kv.second.ptr);
    kv.second.ptr = nullptr;
    kv.second.count = 0;
  }
  delete m;
  ctx->tile_lists = nullptr;
}

void ScreenOperands::setup(const std::vector<int64_t>* phase_rows) {
  ADG_REQUIRE(n <= 65535LL * SC_BN, "evaluate: SCREEN engine supports n <= 8388480");
  T = (n + SC_BN - 1) / SC_BN;
  // rows read by A (256-row blocks) and by B (160-row blocks)
  rows_pad = std::max((n + SC_PM - 1) / SC_PM * SC_PM, T * SC_BN);
  kp = (d + SC_BK - 1) / SC_BK * SC_BK;
  kr = (r + SC_BK - 1) / SC_BK * SC_BK;
  ktot = kp + kr;
  hi.alloc((size_t)(rows_pad * ktot), ctx->stream);
  lo.alloc((size_t)(rows_pad * ktot), ctx->stream);
  meta.alloc((size_t)rows_pad, ctx->stream);
  lo_flag.alloc(1, ctx->stream);
  lo_flag.zero();
  map_a_hi = make_plane_map(hi.ptr, rows_pad, ktot, SC_BM);
  map_a_lo = make_plane_map(lo.ptr, rows_pad, ktot, SC_BM);
  map_b_hi = make_plane_map(hi.ptr, rows_pad, ktot, SC_BNH);
  map_b_lo = make_plane_map(lo.ptr, rows_pad, ktot, SC_BNH);
  static std::mutex cache_mu;
  static std::map<int64_t, std::vector<uint32_t>> cache;  // banded tile lists by (T, band) (host)
  std::vector<uint32_t>* tlp;
  {
    std::lock_guard<std::mutex> lk(cache_mu);
    const int64_t key = n * 4096 + screen_band(ktot);
    auto it = cache.find(key);
    if (it == cache.end()) it = cache.emplace(key, build_tile_list(n, screen_band(ktot))).first;
    tlp = &it->second;
  }
  if (phase_rows) {
    // the phased list is a pure function of (n, band, phase rows): built and
    // uploaded once per context (negative keys: the banded lists' are >= 0)
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) {
      for (int b = 0; b < 8; ++b) h = (h ^ ((v >> (8 * b)) & 0xFF)) * 1099511628211ull;
    };
    mix((uint64_t)n);
    mix((uint64_t)screen_band(ktot));
    for (int64_t v : *phase_rows) mix((uint64_t)v);
    const int64_t key = (int64_t)(h | (1ull << 63));
    struct Phased {
      std::vector<int64_t> rows, end;
      int64_t count;
    };
    static std::map<int64_t, Phased> phased_host;  // under cache_mu
    if (!ctx->tile_lists) ctx->tile_lists = new TileListCache();
    auto& m = *static_cast<TileListCache*>(ctx->tile_lists);
    std::lock_guard<std::mutex> lk(cache_mu);
    auto ph = phased_host.find(key);
    auto it = m.find(key);
    if (ph == phased_host.end() || ph->second.rows != *phase_rows || it == m.end()) {
      std::vector<int64_t> end;
      const std::vector<uint32_t> phased = phase_tiles(*tlp, *phase_rows, end);
      const std::vector<uint32_t> slots = tile_slots(phased, n);
      DevBuf<uint32_t> dl(2 * phased.size(), ctx->stream);  // [tiles | slots]
      ADG_CUDA(cudaMemcpyAsync(dl.ptr, phased.data(), phased.size() * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, ctx->stream));
      ADG_CUDA(cudaMemcpyAsync(dl.ptr + phased.size(), slots.data(), slots.size() * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, ctx->stream));
      // (pageable source: staged before the call returns; the vectors may go)
      phased_host[key] = Phased{*phase_rows, end, (int64_t)phased.size()};
      m[key] = std::move(dl);
      ph = phased_host.find(key);
      it = m.find(key);
    }
    phase_tile_end = ph->second.end;
    num_tiles = ph->second.count;
    tiles_ptr = it->second.ptr;
    slots_ptr = it->second.ptr + num_tiles;
  } else {
    // the banded list is a pure function of T: one device copy per context
    num_tiles = (int64_t)tlp->size();
    if (!ctx->tile_lists) ctx->tile_lists = new TileListCache();
    auto& m = *static_cast<TileListCache*>(ctx->tile_lists);
    const int64_t key = n * 4096 + screen_band(ktot);
    auto it = m.find(key);
    if (it == m.end()) {
      const std::vector<uint32_t> slots = tile_slots(*tlp, n);
      DevBuf<uint32_t> dl(2 * tlp->size(), ctx->stream);  // [tiles | slots]
      ADG_CUDA(cudaMemcpyAsync(dl.ptr, tlp->data(), tlp->size() * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, ctx->stream));
      ADG_CUDA(cudaMemcpyAsync(dl.ptr + tlp->size(), slots.data(), slots.size() * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, ctx->stream));
      // (pageable source: staged before the call returns; `slots` may go)
      it = m.emplace(key, std::move(dl)).first;
    }
    tiles_ptr = it->second.ptr;
    slots_ptr = it->second.ptr + tlp->size();
    // the same tiles as pairs for screen_mc_kernel
    const int64_t mkey = (n * 4096 + screen_band(ktot)) | (1LL << 62);
    auto mt = m.find(mkey);
    if (mt == m.end()) {
      const std::vector<uint32_t> pairs = build_tile_pairs(n, screen_band(ktot));
      std::vector<uint32_t> real;
      real.reserve(pairs.size());
      for (uint32_t e : pairs) real.push_back(e == SC_DUMMY ? 0u : e);
      std::vector<uint32_t> slots = tile_slots(real, n);
      for (size_t q = 0; q < pairs.size(); ++q)
        if (pairs[q] == SC_DUMMY) slots[q] = 0;
      DevBuf<uint32_t> dl(2 * pairs.size(), ctx->stream);  // [entries | slots]
      ADG_CUDA(cudaMemcpyAsync(dl.ptr, pairs.data(), pairs.size() * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, ctx->stream));
      ADG_CUDA(cudaMemcpyAsync(dl.ptr + pairs.size(), slots.data(), slots.size() * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, ctx->stream));
      mt = m.emplace(mkey, std::move(dl)).first;
    }
    mc_pairs = (int64_t)(mt->second.count / 4);
    mc_tiles_ptr = mt->second.ptr;
    mc_slots_ptr = mt->second.ptr + 2 * mc_pairs;
  }
  // Error model (documented in DESIGN.md): each of the 3 * (K/16) MMA
  // accumulation steps may round the fp32 accumulator (<= 2^-24 relative to
  // |x||y| <= (|x|^2+|y|^2)/2), the split drops lo.lo (<= 2^-22), the epilogue
  // adds a handful of fp32 roundings.  eps bounds |o - o_exact| / (|x|^2+|y|^2).
  const int64_t k16 = (d + 15) / 16 + (r + 15) / 16;
  eps = (float)((3.0 * (double)k16 + 64.0) * std::ldexp(1.0, -24));
  tau = (float)(8.0 * eps);
  kc_orig = (int)(kp / SC_BK);
  kc_total = (int)(ktot / SC_BK);
  const int64_t rem_o = d - (kp - SC_BK);
  const int64_t rem_e = r - (kr - SC_BK);
  k16_last_orig = (int)((rem_o + 15) / 16);
  k16_last_emb = (int)((rem_e + 15) / 16);
}

void ScreenOperands::prep_rows(const void* X, adg_dtype xd, const void* Y, adg_dtype yd,
                               const double* mx, const double* my, int64_t row0, int64_t row1) {
  if (row1 > rows_pad) row1 = rows_pad;
  if (row1 <= row0) return;
  const unsigned grid = blocks_for((row1 - row0) * 32, 256);
  ADG_DISPATCH_DTYPE(xd, TO, {
    ADG_DISPATCH_DTYPE(yd, TE, {
      if constexpr (!std::is_same<TO, double>::value && !std::is_same<TE, double>::value) {
        const int64_t kp4 = kp / 4;
        const bool vec = d % 4 == 0 && (reinterpret_cast<uintptr_t>(X) % (4 * sizeof(TO))) == 0 &&
                         kp4 <= 32 * 16;
        const size_t msh = sizeof(float) * (size_t)(((d + 3) & ~3LL) + r);
        auto args = [&](auto kern) {
          if (msh > 48 * 1024) ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msh));
          kern<<<grid, 256, msh, ctx->stream>>>((const TO*)X, n, d, mx, (const TE*)Y, r, my, rows_pad,
                                                kp, ktot, hi.ptr, lo.ptr, meta.ptr, row0, row1, lo_flag.ptr);
        };
        if (vec && kp4 <= 64)
          args(prep_vec_kernel<TO, TE, 2>);
        else if (vec && kp4 <= 128)
          args(prep_vec_kernel<TO, TE, 4>);
        else if (vec && kp4 <= 256)
          args(prep_vec_kernel<TO, TE, 8>);
        else if (vec)
          args(prep_vec_kernel<TO, TE, 16>);
        else
          args(prep_f32_kernel<TO, TE>);
      } else
        prep_kernel<TO, TE><<<grid, 256, 0, ctx->stream>>>((const TO*)X, n, d, mx, (const TE*)Y, r,
                                                           my, rows_pad, kp, ktot, hi.ptr, lo.ptr,
                                                           meta.ptr, row0, row1, lo_flag.ptr);
    });
  });
  after_launch(ctx);
}

ScreenOperands::ScreenOperands(adg_ctx* c, int64_t n_, int64_t d_, int64_t r_,
                               const std::vector<int64_t>* phase_rows)
    : ctx(c), n(n_), d(d_), r(r_) {
  setup(phase_rows);
}

ScreenOperands::ScreenOperands(adg_ctx* c, const void* X, adg_dtype xd, int64_t n_, int64_t d_,
                               const void* Y, adg_dtype yd, int64_t r_)
    : ctx(c), n(n_), d(d_), r(r_) {
  setup(nullptr);
  refresh(X, xd, Y, yd);
}

void ScreenOperands::refresh(const void* X, adg_dtype xd, const void* Y, adg_dtype yd) {
  lo_flag.zero();
  DevBuf<double> mx((size_t)d, ctx->stream), my((size_t)std::max<int64_t>(r, 1), ctx->stream);
  // centring shift for conditioning only (distances are shift-invariant and the
  // error bound uses the shifted norms): mean of <= kShiftRows evenly spaced rows
  screen_shift(ctx, X, xd, n, d, mx.ptr);
  if (r > 0) column_means_sampled(ctx, Y, yd, n, r, kShiftRows, my.ptr);
  prep_rows(X, xd, Y, yd, mx.ptr, my.ptr, 0, rows_pad);
}

// |x|^2 (fp64) of the rows 0, step, 2 step, ... (m of them): one warp per row.
template <typename T>
__global__ void sampled_sqnorm_kernel(const T* __restrict__ X, int64_t m, int64_t d, int64_t step,
                                      double* __restrict__ out) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  double acc = 0.0;
  for (int64_t t = lane; t < d; t += 32) {
    const double v = to_f64(X[w * step * d + t]);
    acc = fma(v, v, acc);
  }
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) out[w] = acc;
}

// Zero the shift when the sampled rows are already nearly centred:
// |mean|^2 <= 3/4 of their mean |x|^2, i.e. centring would shrink the norms
// the error bound scales with by less than 4x.  Fixed-shape reductions:
// the decision is deterministic.
__global__ void shift_rule_kernel(double* __restrict__ mx, int64_t d, const double* __restrict__ qsum,
                                  int64_t m) {
  __shared__ double part[256];
  __shared__ int zero_it;
  double a = 0.0;
  for (int64_t t = threadIdx.x; t < d; t += blockDim.x) a = fma(mx[t], mx[t], a);
  part[threadIdx.x] = a;
  __syncthreads();
  for (int s = blockDim.x / 2; s; s >>= 1) {
    if ((int)threadIdx.x < s) part[threadIdx.x] += part[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) zero_it = part[0] <= 0.75 * (*qsum / (double)(m > 0 ? m : 1));
  __syncthreads();
  if (zero_it)
    for (int64_t t = threadIdx.x; t < d; t += blockDim.x) mx[t] = 0.0;
}

void screen_shift(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d, double* mx) {
  column_means_sampled(ctx, X, xd, n, d, kShiftRows, mx);
  // bf16 rows are exact in the fp16 hi plane only uncentred (x - mean has
  // more significant bits than bf16's 8): when centring buys little, skip it
  // and the screen runs the original side in one MMA pass (ScreenParams::lo_flag)
  if (xd != ADG_BF16 || n == 0 || std::getenv("ADG_SCREEN_KEEP_SHIFT")) return;
  const int64_t step = std::max<int64_t>(1, (n + kShiftRows - 1) / kShiftRows);
  const int64_t m = (n - 1) / step + 1;
  DevBuf<double> q((size_t)m, ctx->stream), qs(1, ctx->stream);
  sampled_sqnorm_kernel<__nv_bfloat16><<<blocks_for(m * 32, 256), 256, 0, ctx->stream>>>(
      static_cast<const __nv_bfloat16*>(X), m, d, step, q.ptr);
  after_launch(ctx);
  ordered_sum(ctx, q.ptr, m, qs.ptr);
  shift_rule_kernel<<<1, 256, 0, ctx->stream>>>(mx, d, qs.ptr, m);
  after_launch(ctx);
}

// Shared memory of screen_kernel: ring, barriers, column metadata, warp sums,
// the per-CTA u32 counters (bins + 1 slots and a trash slot; none when
// global_hist moves them to per-CTA global scratch) and the per-thread /
// per-warp counters of HMODE 1 / 3.
static size_t smem_for(int stages, int bins, int hmode, bool global_hist = false) {
  const size_t nslot = (size_t)bins + 2;
  const size_t base = 1024 /*align slack*/ + (size_t)stages * SC_STAGE_BYTES +
                      (2 * stages + 6) * sizeof(uint64_t) + 16 + 2 * SC_BN * sizeof(float4) +
                      2 * SC_EPI_WARPS * sizeof(double) +
                      (global_hist ? 0 : (size_t)((bins + 5) & ~3) * sizeof(unsigned));
  const size_t hist = hmode == 1   ? nslot * SC_EPI_THREADS                      // u8 per thread
                      : hmode == 3 ? (size_t)SC_EPI_WARPS * nslot * sizeof(unsigned)  // u32 per warp
                                   : 0;
  return base + hist;
}

// Per-thread u8 counters (HMODE 1) with the deepest ring that fits (3 stages
// of 52 KB at 50 bins; a 4th stage -- tried by keeping u8 counters for the low
// bins only -- measured 8 % slower on C3, 2 stages 12 % slower); larger bin
// counts move to per-warp match-aggregated
// counters (HMODE 3: 16 x less shared memory, but MATCH.ANY per pair made C3
// 9 % slower even with a 4th stage), then to shared atomics.
// ADG_SCREEN_HMODE forces a mode (profiling aid).
ScreenConfig screen_config(int bins) {
  const size_t cap = 227 * 1024;
  const char* e = std::getenv("ADG_SCREEN_HMODE");
  const int forced = e ? std::atoi(e) : -1;
  const char* es = std::getenv("ADG_SCREEN_STAGES");  // profiling aid
  const int fst = es ? std::atoi(es) : -1;
  for (int hm : {1, 3})
    for (int st : {4, 3, 2})
      if ((forced < 0 || forced == hm) && (fst < 0 || fst == st) && smem_for(st, bins, hm) <= cap)
        return {st, hm, smem_for(st, bins, hm)};
  for (int st : {4, 3, 2})
    if (smem_for(st, bins, 0) <= cap) return {st, 0, smem_for(st, bins, 0)};
  // more bins than shared memory holds: per-CTA counters in global scratch
  return {4, 0, smem_for(4, bins, 0, true), true};
}

int screen_tile_slots() { return 2; }  // one ordered partial sum per CTA of the pair

// Width of the edge band, in units of the pair's rigorous error bound, for
// an evaluation that bins edge pairs exactly (ADG_ENGINE_SCREEN_EXACT_HIST)
// or not (0: every pair binned from its screened value).  ADG_EDGE_BAND
// overrides both (profiling aid).
double screen_edge_band(bool exact_hist) {
  const char* e = std::getenv("ADG_EDGE_BAND");
  if (e) return std::atof(e);
  return exact_hist ? kScreenEdgeBand : 0.0;
}

void run_screen(adg_ctx* ctx, const ScreenOperands& ops, int64_t tile_begin, int64_t tile_end,
                int bins, double hist_max, const ScreenPartials& out, bool max_only,
                cudaStream_t stream) {
  if (tile_end <= tile_begin) return;
  const bool own = stream == nullptr || stream == ctx->stream;  // (timed with the context's events)
  cudaStream_t st = own ? ctx->stream : stream;
  ScreenParams p;
  p.tiles = ops.tiles_ptr;
  p.tile_begin = tile_begin;
  p.tile_end = tile_end;
  p.tile_slots = ops.slots_ptr;
  p.meta = ops.meta.ptr;
  p.n = (int)ops.n;
  p.kc_orig = ops.kc_orig;
  p.kc_total = ops.kc_total;
  p.k16_last_orig = ops.k16_last_orig;
  p.k16_last_emb = ops.k16_last_emb;
  p.bins = bins;
  p.hist_scale = (float)((double)bins / hist_max);
  p.tau = ops.tau;
  p.eps = ops.eps;
  p.hist = out.hist;
  p.tile_sums = out.tile_sums;
  p.row_max = out.row_max;
  p.row_bound = out.row_bound;
  p.near_pairs = out.near_pairs;
  p.near_count = out.near_count;
  p.near_cap = out.near_cap;
  p.row_tau2 = nullptr;
  p.knn_out = nullptr;
  p.edge_pairs = out.edge_pairs;
  p.edge_count = out.edge_count;
  p.edge_cap = out.edge_cap;
  p.edge_f = out.edge_f;
  p.hist_scratch = nullptr;
  const char* dbg = std::getenv("ADG_SCREEN_DEBUG");
  p.debug = dbg ? std::atoi(dbg) : 0;
  ctx->screen_forced3 = std::getenv("ADG_SCREEN_ORIG3") != nullptr;
  p.lo_flag = ctx->screen_forced3 ? nullptr : ops.lo_flag.ptr;  // ORIG3: always 3 passes
  const ScreenConfig cfg = max_only ? ScreenConfig{4, 2, smem_for(4, 0, 2)} : screen_config(bins);
  const int64_t ntiles = tile_end - tile_begin;
  const unsigned clusters = (unsigned)std::min<int64_t>(ntiles, ctx->num_sms / 2);
  const bool edges = out.edge_f > 0.f && !max_only;
  auto pick = [&](auto mode_tag) {
    constexpr int M = decltype(mode_tag)::value;
    if (edges)
      return cfg.stages == 4   ? screen_kernel<4, M, true>
             : cfg.stages == 3 ? screen_kernel<3, M, true>
                               : screen_kernel<2, M, true>;
    return cfg.stages == 4   ? screen_kernel<4, M>
           : cfg.stages == 3 ? screen_kernel<3, M>
                             : screen_kernel<2, M>;
  };
  auto kern = max_only         ? screen_kernel<4, 2>
              : cfg.hmode == 3 ? pick(std::integral_constant<int, 3>{})
              : cfg.hmode == 1 ? pick(std::integral_constant<int, 1>{})
                               : pick(std::integral_constant<int, 0>{});
  // ADG_SCREEN_MC=1 (experiment, off by default): a full pass over the banded
  // list as 4-CTA clusters sharing A by multicast (screen_mc_kernel).  The
  // report is bit-identical; measured slower on C3 (6.77 against 6.01 ms):
  // 4-CTA clusters pack fewer SMs per GPC, and per SM the halved A requests
  // bought ~2 %.  Shards and pipeline phases use the pairs.
  const char* mce = std::getenv("ADG_SCREEN_MC");
  const bool mc = !max_only && ops.mc_pairs > 0 && tile_begin == 0 && tile_end == ops.num_tiles &&
                  ops.tiles_ptr != nullptr && mce != nullptr && std::atoi(mce) != 0 && ctx->num_sms >= 4;
  if (mc) {
    auto pick_mc = [&](auto mode_tag) {
      constexpr int M = decltype(mode_tag)::value;
      if (edges)
        return cfg.stages == 4   ? screen_mc_kernel<4, M, true>
               : cfg.stages == 3 ? screen_mc_kernel<3, M, true>
                                 : screen_mc_kernel<2, M, true>;
      return cfg.stages == 4   ? screen_mc_kernel<4, M>
             : cfg.stages == 3 ? screen_mc_kernel<3, M>
                               : screen_mc_kernel<2, M>;
    };
    kern = cfg.hmode == 3 ? pick_mc(std::integral_constant<int, 3>{})
           : cfg.hmode == 1 ? pick_mc(std::integral_constant<int, 1>{})
                            : pick_mc(std::integral_constant<int, 0>{});
    p.tiles = ops.mc_tiles_ptr;
    p.tile_slots = ops.mc_slots_ptr;
    p.tile_begin = 0;
    p.tile_end = ops.mc_pairs;
  }
  if (max_only) p.bins = 0;
  DevBuf<unsigned> scratch;
  if (cfg.global_hist && !max_only) {
    scratch.alloc((size_t)(2 * clusters) * (size_t)(bins + 2), st);
    p.hist_scratch = scratch.ptr;  // zeroed by the kernel; freed stream-ordered after it
  }
  ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem));
  if (own) ADG_CUDA(cudaEventRecord(ctx->ev_a, st));
  unsigned grid = 2 * clusters;
  if (mc) {
    // 4-CTA clusters must fit a GPC: launch only as many as can be resident
    // at once (the persistent loop spreads the tile pairs over them)
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(4u * (unsigned)(ctx->num_sms / 4));
    lc.blockDim = dim3(SC_THREADS);
    lc.dynamicSmemBytes = cfg.smem;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 4;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    lc.attrs = &at;
    lc.numAttrs = 1;
    int maxc = 0;
    ADG_CUDA(cudaOccupancyMaxActiveClusters(&maxc, (const void*)kern, &lc));
    ADG_REQUIRE(maxc >= 1, "screen: 4-CTA clusters cannot be resident");
    grid = 4u * (unsigned)std::min<int64_t>(ops.mc_pairs, maxc);
  }
  kern<<<grid, SC_THREADS, cfg.smem, st>>>(ops.map_a_hi, ops.map_a_lo, ops.map_b_hi, ops.map_b_lo, p);
  after_launch(ctx);
  if (own) {
    ADG_CUDA(cudaEventRecord(ctx->ev_b, st));
    ctx->last_screen_ms = -2.0;  // pending: resolved by adg_last_screen_kernel_ms
  }
}

// k-NN candidate pass (HMODE 4) over the whole banded triangle: ops built with
// r = 0 (orig K chunks only); tau2 holds rows_pad radii (0 past n).
void run_screen_knn(adg_ctx* ctx, const ScreenOperands& ops, const float* tau2, uint4* out,
                    unsigned long long* count, long long cap) {
  if (ops.num_tiles <= 0) return;
  ADG_REQUIRE(ops.r == 0, "run_screen_knn: operands must carry no embedding");
  ScreenParams p{};
  p.tiles = ops.tiles_ptr;
  p.tile_begin = 0;
  p.tile_end = ops.num_tiles;
  p.tile_slots = ops.slots_ptr;
  p.meta = ops.meta.ptr;
  p.n = (int)ops.n;
  p.kc_orig = ops.kc_orig;
  p.kc_total = ops.kc_orig;
  p.k16_last_orig = ops.k16_last_orig;
  p.k16_last_emb = ops.k16_last_emb;
  p.bins = 0;
  p.hist_scale = 0.f;
  p.tau = ops.tau;
  p.eps = ops.eps;
  p.near_count = count;
  p.near_cap = cap;
  p.row_tau2 = tau2;
  p.knn_out = out;
  p.debug = 0;
  p.edge_pairs = nullptr;
  p.edge_count = nullptr;
  p.edge_cap = 0;
  p.edge_f = 0.f;
  p.hist_scratch = nullptr;
  p.lo_flag = std::getenv("ADG_SCREEN_ORIG3") ? nullptr : ops.lo_flag.ptr;
  const size_t smem = smem_for(4, 0, 4);
  const unsigned clusters = (unsigned)std::min<int64_t>(ops.num_tiles, ctx->num_sms / 2);
  auto kern = screen_kernel<4, 4>;
  ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<2 * clusters, SC_THREADS, smem, ctx->stream>>>(ops.map_a_hi, ops.map_a_lo, ops.map_b_hi,
                                                        ops.map_b_lo, p);
  after_launch(ctx);
}

}  // namespace adg
