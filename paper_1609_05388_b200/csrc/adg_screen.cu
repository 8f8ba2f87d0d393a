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
//   * the histogram (distortion.cpp:81-87 binning) in per-thread u16 smem
//     counters flushed to global u64,
//   * per-tile partial sums (deterministic slots, ordered reduction later),
//   * per-row screened max and screened max + rigorous error bound, which the
//     exact fp64 refine (adg_exact.cu) uses to recover the reference's max
//     and its lowest (i, j) argmax exactly,
//   * pairs whose screened o is within the noise of 0 (possible duplicates),
//     listed for the exact zero rule of distortion.cpp:66-69.
//
// Kernel structure (one persistent CTA per SM, 320 threads):
//   warp 0     TMA producer: 128x64 fp16 boxes (SWIZZLE_128B) of the hi/lo
//              planes of row block I (A) and J (B) into a 3-stage ring,
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer,
//   warps 2-9  epilogue (two per SM sub-partition; warp w owns TMEM lane
//              quarter w%4 and one 64-column half): tcgen05.ld 32x32b.x32 of
//              the orig / emb accumulators, branch-free pair math.
// TMEM (512 cols) holds two 128x(128+128) accumulator sets, so the epilogue of
// tile t overlaps the MMAs of tile t+1.  Tiles walk the upper triangle of the
// (n/128)^2 block grid in 16-row bands for L2 reuse of both operands.
#include "adg_screen.cuh"

#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>

namespace adg {

// ------------------------------------------------------------ constants
constexpr int SC_BM = 128;           // rows of a tile (TMEM lanes)
constexpr int SC_BN = 128;           // cols of a tile
constexpr int SC_BK = 64;            // fp16 K per stage = one 128-byte swizzle row
constexpr int SC_EPI_WARPS = 8;     // 2 per SM sub-partition, each 32 rows x 64 cols
constexpr int SC_EPI_THREADS = 32 * SC_EPI_WARPS;
constexpr int SC_THREADS = 64 + SC_EPI_THREADS;
constexpr uint32_t SC_OP_BYTES = SC_BM * SC_BK * 2;  // 16 KB per operand plane
constexpr uint32_t SC_STAGE_BYTES = 4 * SC_OP_BYTES; // A_hi, A_lo, B_hi, B_lo
constexpr int SC_FLUSH_TILES = 512;  // u16 private counters: 512 * 64 pairs < 65536
constexpr int SC_BAND = 16;          // tile-list band height (L2 locality)

struct ScreenParams {
  const uint32_t* tiles;  // (I << 16) | J
  int64_t tile_begin, tile_end;
  const float4* meta;  // per padded row: |x|^2, |f|^2, 2^-e, 2^-e'
  int n;
  int kc_orig, kc_total;     // K chunks (of 64) for orig, orig+emb
  int k16_last_orig, k16_last_emb;
  int bins;
  float hist_scale;  // bins / hist_max
  float tau;         // near-zero threshold relative to |x|^2+|y|^2
  float eps;         // error-bound coefficient
  unsigned long long* hist;
  double* tile_sums;
  float* row_max;
  float* row_bound;
  uint32_t* near_pairs;
  unsigned long long* near_count;
  long long near_cap;
};

// ----------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

#define TMEM_LD32(taddr, r)                                                                     \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"       \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),     \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),             \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),          \
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),          \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),          \
        "=r"(r[31])                                                                             \
      : "r"(taddr))

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm_100 format:
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major), SBO>>4
// [32,46) = 1024 B between 8-row core groups, version 1 [46,48), layout
// SWIZZLE_128B = 2 at [61,64)).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor: D=f32, A=B=f16, K-major both, N=128, M=128.
constexpr uint32_t SC_IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(SC_BN >> 3) << 17) |
                              ((uint32_t)(SC_BM >> 4) << 24);

__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_rsqrt(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------------------- the kernel
// Epilogue work for one 32-column chunk of one row (this thread's TMEM lane).
// Branch-free over the 32 pairs: pairs that must not be counted (outside the
// upper triangle / beyond n on edge tiles, or screened as near-coincident)
// contribute v = 0 and are corrected after the loop from two bit masks.
struct EpiRow {
  float rn, rm, ra2, rb2;  // |x_i|^2, |f_i|^2, -2 * 2^-e_i, -2 * 2^-e'_i
  float vmax, umax;
  int i;
};

template <bool EDGE, bool PRIVATE_HIST>
__device__ __forceinline__ void epi_chunk(const uint32_t* g, const uint32_t* h,
                                          const float4* __restrict__ cmeta, uint16_t* __restrict__ hrow,
                                          unsigned* __restrict__ h32,
                                          EpiRow& R, float& tsum, int jbase, int n, float tau, float eps,
                                          float hbias, float hcap, uint32_t& excl_mask,
                                          uint32_t& near_mask) {
  uint32_t excl = 0, nearm = 0;
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) {
    const float4 cm = cmeta[jj];
    const float sn = R.rn + cm.x;
    const float o = fmaf(R.ra2 * cm.z, __uint_as_float(g[jj]), sn);
    const float sm = R.rm + cm.y;
    const float e = fmaf(R.rb2 * cm.w, __uint_as_float(h[jj]), sm);
    const float ro = fast_rcp(o);
    const float q = fmaxf(e * ro, 1e-30f);
    const float rq = fast_rsqrt(q);
    const float v = fabsf(fmaf(q, rq, -1.0f));
    const float t = fmaf(q, sn, sm) * ro;
    const float ub = fmaf(eps * t, rq, v);
    bool skip = !(o > tau * sn);
    if (skip) nearm |= 1u << jj;
    if (EDGE) {
      const int j = jbase + jj;
      const bool valid = (j > R.i) && (j < n) && (R.i < n);
      if (!valid) nearm &= ~(1u << jj);
      skip = skip || !valid;
    }
    if (skip) excl |= 1u << jj;
    const float ve = skip ? 0.0f : v;
    R.vmax = fmaxf(R.vmax, ve);
    R.umax = fmaxf(R.umax, skip ? 0.0f : ub);
    tsum += ve;
    // bin = min(floor(v * bins / hist_max), bins): a round-toward-zero FMA onto
    // 2^23 leaves floor(v * scale) in the low mantissa bits (no F2I needed).
    const float bf = fminf(__fmaf_rz(ve, hbias, 8388608.0f), hcap);
    const int bin = __float_as_int(bf) - 0x4B000000;
    if (PRIVATE_HIST)
      hrow[bin * SC_EPI_THREADS] += 1;
    else
      atomicAdd(&h32[bin], 1u);
  }
  excl_mask = excl;
  near_mask = nearm;
}

template <int SC_STAGES, bool PRIVATE_HIST>
__global__ void __launch_bounds__(SC_THREADS, 1)
screen_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
              const ScreenParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // Carve by byte offsets from the __shared__ array so every access below
  // compiles to LDS/STS (no generic addressing); the ring is 1024-aligned.
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* ring = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + SC_STAGES * SC_STAGE_BYTES);
  uint64_t* full = bars;                   // [STAGES]
  uint64_t* empty = bars + SC_STAGES;      // [STAGES]
  uint64_t* tfull = bars + 2 * SC_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float4* colmeta = reinterpret_cast<float4*>(tmem_slot + 4);  // [2][128]
  uint16_t* h16 = reinterpret_cast<uint16_t*>(colmeta + 2 * SC_BN);  // [bins+1][256]
  unsigned* h32 = reinterpret_cast<unsigned*>(colmeta + 2 * SC_BN);  // [bins+1]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SC_STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), SC_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp >= 2) {
    const int et = threadIdx.x - 64;
    if (PRIVATE_HIST) {
      for (int b = 0; b <= p.bins; ++b) h16[b * SC_EPI_THREADS + et] = 0;
    } else {
      for (int b = et; b <= p.bins; b += SC_EPI_THREADS) h32[b] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_hi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_lo)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = p.tile_begin + blockIdx.x; t < p.tile_end; t += gridDim.x) {
        const uint32_t tij = p.tiles[t];
        const int I = (int)(tij >> 16), J = (int)(tij & 0xFFFF);
        for (int kc = 0; kc < p.kc_total; ++kc) {
          const uint32_t eb = smem_u32(&empty[stage]);
          while (!mbar_try_wait(eb, phase ^ 1)) __nanosleep(32);
          const uint32_t fb = smem_u32(&full[stage]);
          mbar_expect_tx(fb, SC_STAGE_BYTES);
          const uint32_t sbase = smem_u32(ring + stage * SC_STAGE_BYTES);
          tma_load_2d(sbase + 0 * SC_OP_BYTES, &map_hi, fb, kc * SC_BK, I * SC_BM);
          tma_load_2d(sbase + 1 * SC_OP_BYTES, &map_lo, fb, kc * SC_BK, I * SC_BM);
          tma_load_2d(sbase + 2 * SC_OP_BYTES, &map_hi, fb, kc * SC_BK, J * SC_BN);
          tma_load_2d(sbase + 3 * SC_OP_BYTES, &map_lo, fb, kc * SC_BK, J * SC_BN);
          if (++stage == SC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =========================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t lt = 0;
      for (int64_t t = p.tile_begin + blockIdx.x; t < p.tile_end; t += gridDim.x, ++lt) {
        const int b = (int)(lt & 1);
        const uint32_t use = (uint32_t)(lt >> 1);
        mbar_wait(smem_u32(&tempty[b]), (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_orig = tmem_base + (uint32_t)(b * 256);
        const uint32_t d_emb = d_orig + 128;
        for (int kc = 0; kc < p.kc_total; ++kc) {
          mbar_wait(smem_u32(&full[stage]), phase);
          tc_fence_after();
          const bool is_emb = kc >= p.kc_orig;
          const uint32_t dacc = is_emb ? d_emb : d_orig;
          const bool first = (kc == 0) || (kc == p.kc_orig);
          const int nk = (kc == p.kc_orig - 1) ? p.k16_last_orig
                                                : ((kc == p.kc_total - 1) ? p.k16_last_emb : 4);
          const uint32_t sbase = smem_u32(ring + stage * SC_STAGE_BYTES);
          for (int k = 0; k < nk; ++k) {
            const uint32_t koff = (uint32_t)(k * 32);  // 16 fp16 = 32 bytes along K
            const uint64_t a_hi = sw128_desc(sbase + 0 * SC_OP_BYTES + koff);
            const uint64_t a_lo = sw128_desc(sbase + 1 * SC_OP_BYTES + koff);
            const uint64_t b_hi = sw128_desc(sbase + 2 * SC_OP_BYTES + koff);
            const uint64_t b_lo = sw128_desc(sbase + 3 * SC_OP_BYTES + koff);
            tc_mma_f16(dacc, a_hi, b_hi, SC_IDESC, (first && k == 0) ? 0u : 1u);
            tc_mma_f16(dacc, a_hi, b_lo, SC_IDESC, 1u);
            tc_mma_f16(dacc, a_lo, b_hi, SC_IDESC, 1u);
          }
          tc_commit(smem_u32(&empty[stage]));  // frees the smem slot when these MMAs finish
          if (++stage == SC_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(smem_u32(&tfull[b]));  // accumulators of this tile are ready
      }
    }
  } else {
    // ======================= epilogue (warps 2..9) ==============
    const int et = threadIdx.x - 64;            // 0..255
    const int quarter = warp & 3;               // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;           // column half [64*half, 64*half + 64)
    const int row_in_tile = quarter * 32 + lane;
    uint16_t* hrow = h16 + et;                  // this thread's private counters (stride 256)
    const int bins = p.bins;
    const float tau = p.tau, eps = p.eps;
    const float hbias = p.hist_scale;
    const float hcap = 8388608.0f + (float)bins;
    int64_t lt = 0;
    for (int64_t t = p.tile_begin + blockIdx.x; t < p.tile_end; t += gridDim.x, ++lt) {
      const int b = (int)(lt & 1);
      const uint32_t use = (uint32_t)(lt >> 1);
      const uint32_t tij = p.tiles[t];
      const int I = (int)(tij >> 16), J = (int)(tij & 0xFFFF);
      if (et < SC_BN) colmeta[b * SC_BN + et] = p.meta[(int64_t)J * SC_BN + et];
      asm volatile("bar.sync 1, %0;" ::"n"(SC_EPI_THREADS) : "memory");
      EpiRow R;
      R.i = I * SC_BM + row_in_tile;
      {
        const float4 rmeta = p.meta[R.i];
        R.rn = rmeta.x;
        R.rm = rmeta.y;
        R.ra2 = -2.0f * rmeta.z;
        R.rb2 = -2.0f * rmeta.w;
      }
      R.vmax = 0.0f;
      R.umax = 0.0f;
      const bool edge = (I == J) || ((J + 1) * SC_BN > p.n) || ((I + 1) * SC_BM > p.n);
      mbar_wait(smem_u32(&tfull[b]), use & 1);
      tc_fence_after();
      double dsum = 0.0;
      const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * 256);
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int col0 = half * 64 + c * 32;
        uint32_t g[32], h[32];
        TMEM_LD32(lane_base + (uint32_t)col0, g);
        TMEM_LD32(lane_base + 128u + (uint32_t)col0, h);
        tmem_ld_wait();
        if (c == 1) {
          // both chunks of this warp are in registers: release the TMEM buffer early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&tempty[b]));
        }
        float tsum = 0.0f;
        uint32_t excl, nearm;
        const float4* cmeta = colmeta + b * SC_BN + col0;
        const int jbase = J * SC_BN + col0;
        if (edge)
          epi_chunk<true, PRIVATE_HIST>(g, h, cmeta, hrow, h32, R, tsum, jbase, p.n, tau, eps,
                                        hbias, hcap, excl, nearm);
        else
          epi_chunk<false, PRIVATE_HIST>(g, h, cmeta, hrow, h32, R, tsum, jbase, p.n, tau, eps,
                                         hbias, hcap, excl, nearm);
        dsum += (double)tsum;
        if (excl) {
          // excluded pairs were binned as 0: take them back out
          if (PRIVATE_HIST)
            hrow[0] = (uint16_t)(hrow[0] - __popc(excl));
          else
            atomicSub(&h32[0], (unsigned)__popc(excl));
          while (nearm) {
            const int jj = __ffs(nearm) - 1;
            nearm &= nearm - 1;
            const unsigned long long slot = atomicAdd(p.near_count, 1ull);
            if ((long long)slot < p.near_cap) {
              p.near_pairs[2 * slot] = (uint32_t)R.i;
              p.near_pairs[2 * slot + 1] = (uint32_t)(jbase + jj);
            }
          }
        }
      }
      if (R.i < p.n) {
        if (R.vmax > 0.0f) atomicMax(reinterpret_cast<int*>(p.row_max) + R.i, __float_as_int(R.vmax));
        if (R.umax > 0.0f) atomicMax(reinterpret_cast<int*>(p.row_bound) + R.i, __float_as_int(R.umax));
      }
#pragma unroll
      for (int s = 16; s; s >>= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, s);
      if (lane == 0) p.tile_sums[t * SC_EPI_WARPS + (warp - 2)] = dsum;
      if (PRIVATE_HIST && ((lt + 1) % SC_FLUSH_TILES) == 0) {
        for (int bb = 0; bb <= bins; ++bb) {
          const unsigned cnt = hrow[bb * SC_EPI_THREADS];
          if (cnt) {
            atomicAdd(&p.hist[bb], (unsigned long long)cnt);
            hrow[bb * SC_EPI_THREADS] = 0;
          }
        }
      }
    }
    if (PRIVATE_HIST) {
      for (int bb = 0; bb <= bins; ++bb) {
        const unsigned cnt = hrow[bb * SC_EPI_THREADS];
        if (cnt) atomicAdd(&p.hist[bb], (unsigned long long)cnt);
      }
    } else {
      asm volatile("bar.sync 1, %0;" ::"n"(SC_EPI_THREADS) : "memory");
      for (int bb = et; bb <= bins; bb += SC_EPI_THREADS)
        if (h32[bb]) atomicAdd(&p.hist[bb], (unsigned long long)h32[bb]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
}

// ------------------------------------------------------------ prep kernel
// One warp per padded row: centre (fp64), pick the power-of-two scale, write
// the hi/lo fp16 planes ([rows_pad][ktot], orig at [0,d), emb at [kp, kp+r)),
// and the row metadata computed from the represented value hi+lo.
template <typename TO, typename TE>
__global__ void prep_kernel(const TO* __restrict__ X, int64_t n, int64_t d,
                            const double* __restrict__ mx, const TE* __restrict__ Y, int64_t r,
                            const double* __restrict__ my, int64_t rows_pad, int64_t kp,
                            int64_t ktot, __half* __restrict__ hi, __half* __restrict__ lo,
                            float4* __restrict__ meta) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows_pad) return;
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
  if (lane == 0) meta[row] = m4;
}

// ----------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    ADG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess)
      fail(ADG_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

static CUtensorMap make_plane_map(const __half* base, int64_t rows, int64_t ktot) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)ktot, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ktot * 2)};
  cuuint32_t box[2] = {(cuuint32_t)SC_BK, (cuuint32_t)SC_BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult rc = get_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)base, dims, strides,
                                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) fail(ADG_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)rc));
  return m;
}

// Banded upper-triangle order: for each band of SC_BAND row blocks, walk the
// column blocks J >= band start and, for each, the band's rows I <= J.
std::vector<uint32_t> build_tile_list(int64_t T) {
  std::vector<uint32_t> tiles;
  tiles.reserve((size_t)(T * (T + 1) / 2));
  for (int64_t I0 = 0; I0 < T; I0 += SC_BAND) {
    const int64_t I1 = std::min<int64_t>(I0 + SC_BAND, T);
    for (int64_t J = I0; J < T; ++J)
      for (int64_t I = I0; I < I1 && I <= J; ++I)
        tiles.push_back((uint32_t)((I << 16) | J));
  }
  return tiles;
}

ScreenOperands::ScreenOperands(adg_ctx* c, const void* X, adg_dtype xd, int64_t n_, int64_t d_,
                               const void* Y, adg_dtype yd, int64_t r_)
    : ctx(c), n(n_), d(d_), r(r_) {
  ADG_REQUIRE(n <= 65535LL * SC_BM, "evaluate: SCREEN engine supports n <= 8388480");
  T = (n + SC_BM - 1) / SC_BM;
  rows_pad = T * SC_BM;
  kp = (d + SC_BK - 1) / SC_BK * SC_BK;
  kr = (r + SC_BK - 1) / SC_BK * SC_BK;
  ktot = kp + kr;
  DevBuf<double> mx((size_t)d, ctx->stream), my((size_t)r, ctx->stream);
  column_means(ctx, X, xd, n, d, mx.ptr);
  column_means(ctx, Y, yd, n, r, my.ptr);
  hi.alloc((size_t)(rows_pad * ktot), ctx->stream);
  lo.alloc((size_t)(rows_pad * ktot), ctx->stream);
  meta.alloc((size_t)rows_pad, ctx->stream);
  ADG_DISPATCH_DTYPE(xd, TO, {
    ADG_DISPATCH_DTYPE(yd, TE, {
      prep_kernel<TO, TE><<<blocks_for(rows_pad * 32, 256), 256, 0, ctx->stream>>>(
          (const TO*)X, n, d, mx.ptr, (const TE*)Y, r, my.ptr, rows_pad, kp, ktot, hi.ptr, lo.ptr,
          meta.ptr);
    });
  });
  after_launch(ctx);
  map_hi = make_plane_map(hi.ptr, rows_pad, ktot);
  map_lo = make_plane_map(lo.ptr, rows_pad, ktot);
  static std::mutex cache_mu;
  static std::map<int64_t, std::vector<uint32_t>> cache;  // tile lists by T (host)
  std::vector<uint32_t>* tlp;
  {
    std::lock_guard<std::mutex> lk(cache_mu);
    auto it = cache.find(T);
    if (it == cache.end()) it = cache.emplace(T, build_tile_list(T)).first;
    tlp = &it->second;
  }
  const std::vector<uint32_t>& tl = *tlp;
  num_tiles = (int64_t)tl.size();
  tiles.alloc(tl.size(), ctx->stream);
  ADG_CUDA(cudaMemcpyAsync(tiles.ptr, tl.data(), tl.size() * sizeof(uint32_t),
                           cudaMemcpyHostToDevice, ctx->stream));
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

static size_t smem_for(int stages, int bins, bool priv) {
  const size_t base = 1024 /*align slack*/ + (size_t)stages * SC_STAGE_BYTES +
                      (2 * stages + 4) * sizeof(uint64_t) + 16 + 2 * SC_BN * sizeof(float4);
  return base + (priv ? (size_t)(bins + 1) * SC_EPI_THREADS * sizeof(uint16_t)
                      : (size_t)(bins + 1) * sizeof(unsigned));
}

// Pick the deepest ring that still leaves room for per-thread u16 histogram
// counters; very large bin counts fall back to shared atomics.
ScreenConfig screen_config(int bins) {
  const size_t cap = 227 * 1024;
  if (smem_for(3, bins, true) <= cap) return {3, true, smem_for(3, bins, true)};
  if (smem_for(2, bins, true) <= cap) return {2, true, smem_for(2, bins, true)};
  return {3, false, smem_for(3, bins, false)};
}

int screen_tile_slots() { return SC_EPI_WARPS; }

void run_screen(adg_ctx* ctx, const ScreenOperands& ops, int64_t tile_begin, int64_t tile_end,
                int bins, double hist_max, const ScreenPartials& out) {
  if (tile_end <= tile_begin) return;
  ScreenParams p;
  p.tiles = ops.tiles.ptr;
  p.tile_begin = tile_begin;
  p.tile_end = tile_end;
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
  const ScreenConfig cfg = screen_config(bins);
  const size_t smem = cfg.smem;
  const int64_t ntiles = tile_end - tile_begin;
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, ctx->num_sms);
  auto kern = cfg.stages == 3 ? (cfg.private_hist ? screen_kernel<3, true> : screen_kernel<3, false>)
                              : screen_kernel<2, true>;
  ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ADG_CUDA(cudaEventRecord(ctx->ev_a, ctx->stream));
  kern<<<grid, SC_THREADS, smem, ctx->stream>>>(ops.map_hi, ops.map_lo, p);
  after_launch(ctx);
  ADG_CUDA(cudaEventRecord(ctx->ev_b, ctx->stream));
  ctx->last_screen_ms = -2.0;  // pending: resolved by adg_last_screen_kernel_ms
}

}  // namespace adg
