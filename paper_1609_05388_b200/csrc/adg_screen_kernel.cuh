// adg_screen_kernel.cuh -- device side of the SCREEN engine (see adg_screen.cu
// for the algorithm and error model).  Included once, by adg_screen.cu.
//
// Persistent 2-CTA clusters (one CTA per SM, 576 threads), cta_group::2 MMAs
// of M=256 x N=160: a pair tile is 256 rows (128 per CTA, its own A operand)
// x 160 columns (B split 80 + 80 across the pair).
//   warp 0      TMA producer (both CTAs): 128x64 A boxes and 80x64 B boxes of
//               the hi/lo planes (SWIZZLE_128B) into a ring of 52 KB stages,
//               completing on the leader CTA's barrier,
//   warp 1      TMEM allocator (cta_group::2); in the leader one thread issues
//               tcgen05.mma.cta_group::2 for the pair and multicasts commits,
//   warps 2-17  epilogue, four per SM sub-partition: warp w owns TMEM lane
//               quarter w%4 and 40 columns of the tile; tcgen05.ld 32x32b of
//               the orig / emb accumulators and branch-free pair math
//               (2 MUFU per pair).
// TMEM (512 cols): two 160-column orig accumulators (double-buffered, so the
// epilogue of tile t overlaps the MMAs of tile t+1) and one 160-column
// embedding accumulator.  screen_mc_kernel (an off-by-default experiment) runs
// the same body as 4-CTA clusters whose two pairs share A by multicast.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdint>

namespace adg {

constexpr int SC_BM = 128;           // rows per CTA (TMEM lanes); 256 per pair
constexpr int SC_PM = 2 * SC_BM;     // rows per pair tile
constexpr int SC_BN = 160;           // cols per pair tile (TMEM: 2 x 160 orig + 160 emb columns)
constexpr int SC_BNH = SC_BN / 2;    // B rows loaded by each CTA
constexpr int SC_BK = 64;            // fp16 K per stage = one 128-byte swizzle row
constexpr int SC_K16 = SC_BK / 16;   // MMA K steps per stage
constexpr int SC_EPI_WARPS = 16;     // 4 per SM sub-partition, 32 rows x 32 cols each
constexpr int SC_EPI_THREADS = 32 * SC_EPI_WARPS;
constexpr int SC_THREADS = 64 + SC_EPI_THREADS;
constexpr int SC_COLS_PER_WARP = SC_BN / (SC_EPI_WARPS / 4);
constexpr uint32_t SC_A_BYTES = SC_BM * SC_BK * 2;    // 16 KB per A plane
constexpr uint32_t SC_B_BYTES = SC_BNH * SC_BK * 2;   // 8 KB per B half-plane
constexpr uint32_t SC_STAGE_BYTES = 2 * SC_A_BYTES + 2 * SC_B_BYTES;  // 48 KB per CTA
constexpr int SC_FLUSH_TILES = 255 / SC_COLS_PER_WARP;  // u8 private counters never wrap
constexpr int SC_GFLUSH_TILES = 1024;  // per-CTA u32 histogram -> global (< 2^25 pairs between)
constexpr int SC_BAND = 32;          // pair-tile bands of 32 x 256 rows (A band L2-resident; B re-read T2/32 times)
constexpr uint32_t SC_PEER_MASK = 0xFEFFFFFFu;  // shared::cluster address of the leader CTA

struct ScreenParams {
  const uint32_t* tiles;  // (I2 << 16) | J  (I2: 256-row block, J: 128-col block)
  int64_t tile_begin, tile_end;
  const uint32_t* tile_slots;  // canonical slot of each listed tile (order-independent sums)
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
  // HMODE 4 (k-NN candidates): per padded row tau_i^2 (an upper bound on the
  // squared k-th neighbour distance); every pair whose screened lower bound
  // reaches a side's radius is written as {query, candidate, lo, hi} to knn_out
  // (slot from near_count, capacity near_cap)
  const float* row_tau2;
  uint4* knn_out;
  // nullptr, or a device flag the prep kernels set when any original-side lo
  // plane entry is non-zero.  Still 0 at launch: every row this launch reads
  // is exactly its fp16 hi plane (e.g. bf16 input), so the original K chunks
  // need one MMA pass (hi.hi; the hi.lo / lo.hi products are exact zeros) and
  // no lo boxes -- the same accumulators, a third of the tensor work.
  const int* lo_flag;
  // Histogram edges: a pair whose screened interval v -/+ edge_f * (ub - v)
  // reaches past a bin edge is not counted; its (i, j) goes to edge_pairs
  // (warp-reserved chunks; unused slots keep the 0xFF sentinel) and the
  // exact fp64 re-binning (adg_exact.cu, edge_bin) counts it.
  uint2* edge_pairs;
  unsigned long long* edge_count;
  long long edge_cap;
  float edge_f;
  // nullptr, or per-CTA global u32 histograms of bins + 2 entries (HMODE 0
  // when the bin counters do not fit in shared memory)
  unsigned* hist_scratch;
  int debug;  // profiling only (ADG_SCREEN_DEBUG): 1 no pair math, 2 no MMA, 3 TMA only, 4 MMA only,
             // 5 A operand loaded every other tile, 6 A always row block 0 (results wrong;
             // traffic/power probes)
};

// ----------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// arrive on the barrier at the same offset in CTA `rank` of the cluster.
// Default semantics (release at CTA scope): the epilogue's TMEM reads are
// complete (tcgen05.wait::ld) and ordered by tcgen05.fence::before_thread_sync,
// so no cluster-scope release fence (MEMBAR.GPU + ERRBAR per arrive) is needed.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(rank));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
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
#ifdef ADG_DEVICE_CHECKS
  unsigned long long spins = 0;
  while (!mbar_try_wait(bar, parity)) ADG_DCHECK(++spins < ADG_WAIT_LIMIT);
#else
  while (!mbar_try_wait(bar, parity)) {
  }
#endif
}

// 2-SM TMA: bytes land in this CTA's smem, completion is counted on the
// leader CTA's barrier (peer bit cleared), as for cta_group::2 operands.
__device__ __forceinline__ void tma_load_2d_2sm(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & SC_PEER_MASK), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// commit the leader's issued MMAs to the barrier at `bar` in the CTAs of `mask`
__device__ __forceinline__ void tc_commit_mask(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}
// 2-SM TMA multicast to the CTAs of `mask` (same shared-memory offset in each);
// each destination pair's leader barrier counts the bytes landing in that pair
__device__ __forceinline__ void tma_load_2d_2sm_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                   int x, int y, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & SC_PEER_MASK), "r"(x), "r"(y), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_mma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

#define TMEM_LD16(taddr, r)                                                                 \
  asm volatile(                                                                               \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15}, [%16];"                                                                      \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),   \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),           \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                                                 \
      : "r"(taddr))

#define TMEM_LD8(taddr, r)                                                                    \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"           \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), \
                 "=r"(r[7])                                                                     \
               : "r"(taddr))

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm_100 format:
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major), SBO>>4
// [32,46) = 1024 B between 8-row core groups, version 1 [46,48), layout type
// SWIZZLE_128B = 2 at [61,64)).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor: D=f32, A=B=f16, K-major both, N=128, M=256 (pair).
constexpr uint32_t SC_IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(SC_BN >> 3) << 17) |
                              ((uint32_t)(SC_PM >> 4) << 24);

// One K16 step of the split product: hi.hi (+ accumulate flag), hi.lo, lo.hi
// -- one asm block so the single issuing lane pays one issue wrapper, not three.
// hi.hi keeps A_hi in the tensor core's A collector (collector::a::fill) and
// hi.lo reuses it (lastuse): A_hi is read from shared memory once, not twice,
// cutting the step's operand reads from 3 (A + B) to 2 A + 3 B.
__device__ __forceinline__ void tc_mma3_f16_pair(uint32_t d_tmem, uint64_t a_hi, uint64_t a_lo,
                                                 uint64_t b_hi, uint64_t b_lo, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "setp.eq.b32 q, %6, %6;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16.collector::a::fill [%0], %1, %3, %5, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16.collector::a::lastuse [%0], %1, %4, %5, q;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, q;\n\t}\n" ::"r"(d_tmem),
      "l"(a_hi), "l"(a_lo), "l"(b_hi), "l"(b_lo), "r"(SC_IDESC), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ int ld_volatile_s32(const int* p) {
  int v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

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

// ------------------------------------------------------------- epilogue
struct EpiRow {
  float rn, rm, ra2, rb2;  // |x_i|^2, |f_i|^2, -2 * 2^-e_i, -2 * 2^-e'_i
  float vmax, umax;
  int i;
};

// 16 pairs (i, jbase..jbase+15) of this thread's row, branch-free: pairs that
// must not be counted (outside the upper triangle / beyond n on edge tiles,
// screened as near-coincident, or -- EDGES -- too close to a bin edge to bin
// from the screened value) contribute v = 0 to the maxima; they are binned as
// 0 and taken back out per tile (excl), or with EDGES land in the trash
// counter (bin index bins + 1, never flushed).
//
//   o = |x_i|^2 + |x_j|^2 - 2 a_i a_j g,   e likewise,   w = (o e)^(-1/2)
//   v = |sqrt(e/o) - 1| = |e - o| / (o + sqrt(o e))   (e - o exact near q=1)
//   bound: |q*/q - 1| <= delta = eps (sn/o + sm/e) = eps (sn e + sm o) w^2,
//          |v* - v| <= sqrt(q) delta <= (1 + v) delta =: t.
// The bin is floor(x * bins / hist_max) capped at bins (distortion.cpp:81-87)
// of x = v + edge_f t and of x = max(v - edge_f t, 0); when the two differ the pair
// goes to the edge list (exact fp64 binning after the screen).
// HMODE: 0 shared-atomic histogram, 1 private u8 counters, 2 max only (no
// histogram, no sums: the max_distortion / sweep probes), 3 per-warp u32
// counters updated by the leader of each group of lanes holding the same bin
// (__match_any_sync; groups have distinct bins, so no atomics) -- 3.3 KB of
// shared memory instead of the u8 counters' 26 KB, which buys a 4th stage.
template <bool EDGE, int HMODE, int NP, bool EDGES>
__device__ __forceinline__ void epi_pairs(const uint32_t* g, const uint32_t* h,
                                          const float4* __restrict__ cmeta,
                                          uint8_t* __restrict__ hrow, unsigned* __restrict__ h32,
                                          EpiRow& R, float& tsum, int jbase, int n, float tau,
                                          float eps, float hbias, float hcap, float ef,
                                          uint64_t& edgem, uint64_t& nearm, uint64_t& excl,
                                          int shift) {
#pragma unroll
  for (int jj = 0; jj < NP; ++jj) {
    const float4 cm = cmeta[jj];
    const float sn = R.rn + cm.x;
    const float o = fmaf(R.ra2 * cm.z, __uint_as_float(g[jj]), sn);
    const float sm = R.rm + cm.y;
    const float e = fmaf(R.rb2 * cm.w, __uint_as_float(h[jj]), sm);
    const float oe = fmaxf(o * e, 1e-37f);
    const float w = fast_rsqrt(oe);
    const float v = fabsf(e - o) * fast_rcp(fmaf(oe, w, o));
    const float c = fmaf(sn, e, sm * o);
    if constexpr (!EDGES) {
      const float ub = fmaf(eps * (c * w) * w, 1.0f + v, v);
      bool skip = !(o > tau * sn);
      const uint64_t bit = 1ull << (jj + shift);
      if (skip) nearm |= bit;
      if (EDGE) {
        const int j = jbase + jj;
        const bool valid = (j > R.i) && (j < n) && (R.i < n);
        if (!valid) nearm &= ~bit;
        skip = skip || !valid;
      }
      if (skip) excl |= bit;
      const float ve = skip ? 0.0f : v;
      R.vmax = fmaxf(R.vmax, ve);
      R.umax = fmaxf(R.umax, skip ? 0.0f : ub);
      if constexpr (HMODE != 2) {
        tsum += ve;
        // floor(v * bins / hist_max) capped at bins: a round-toward-zero FMA
        // onto 2^23 leaves it in the low mantissa bits (no F2I needed);
        // skipped pairs (ve = 0) land in bin 0 and are taken back out per tile
        const float bf = fminf(__fmaf_rz(ve, hbias, 8388608.0f), hcap);
        const int bin = __float_as_int(bf) - 0x4B000000;
        ADG_DCHECK(bin >= 0 && bin <= (int)(hcap - 8388608.0f) + 1);
        if constexpr (HMODE == 1) {
          hrow[bin * SC_EPI_THREADS] += 1;
        } else if constexpr (HMODE == 3) {
          const unsigned grp = __match_any_sync(0xffffffffu, bin);
          if ((int)__ffs(grp) - 1 == (int)(threadIdx.x & 31)) h32[bin] += (unsigned)__popc(grp);
        } else {
          atomicAdd(&h32[bin], 1u);
        }
      }
    } else {
      const float q = eps * (c * w) * w;
      const float t = fmaf(q, v, q);  // (1 + v) delta
      const float ub = v + t;
      bool skip = !(o > tau * sn);
      const uint64_t bit = 1ull << (jj + shift);
      if (skip) nearm |= bit;
      if (EDGE) {
        const int j = jbase + jj;
        const bool valid = (j > R.i) && (j < n) && (R.i < n);
        if (!valid) nearm &= ~bit;
        skip = skip || !valid;
      }
      const float ve = skip ? 0.0f : v;
      R.vmax = fmaxf(R.vmax, ve);
      R.umax = fmaxf(R.umax, skip ? 0.0f : ub);
      if constexpr (HMODE != 2) {
        tsum += ve;
        // bins of v + edge_f t and max(v - edge_f t, 0); a pair whose two bins
        // differ goes to the edge list, skipped and edge pairs to the trash slot
        const float tf = t * ef;
        const float bh = fminf(__fmaf_rz(v + tf, hbias, 8388608.0f), hcap);
        const float bl = fminf(__fmaf_rz(fmaxf(v - tf, 0.0f), hbias, 8388608.0f), hcap);
        const bool unc = bh != bl;
        if (unc && !skip) edgem |= bit;
        const int bin = (skip || unc) ? __float_as_int(hcap) + 1 - 0x4B000000
                                      : __float_as_int(bh) - 0x4B000000;
        ADG_DCHECK(bin >= 0 && bin <= (int)(hcap - 8388608.0f) + 1);
        if constexpr (HMODE == 1) {
          hrow[bin * SC_EPI_THREADS] += 1;
        } else if constexpr (HMODE == 3) {
          const unsigned grp = __match_any_sync(0xffffffffu, bin);
          if ((int)__ffs(grp) - 1 == (int)(threadIdx.x & 31)) h32[bin] += (unsigned)__popc(grp);
        } else {
          atomicAdd(&h32[bin], 1u);
        }
      }
    }
  }
}

// Warp-aggregated append of this thread's edge pairs (bits of `mask` are
// columns jbase + b) into chunks the warp reserves with one atomic; the
// unused tail of a chunk is filled with the 0xFFFFFFFF sentinel when the warp
// moves on (or finishes), so the list needs no initialisation.
struct EdgeChunk {
  unsigned long long base;
  int used, cap;
};
constexpr int SC_EDGE_CHUNK = 128;

__device__ __forceinline__ void seal_edges(const EdgeChunk& ch, const ScreenParams& p, int lane) {
  for (int k = ch.used + lane; k < ch.cap; k += 32) {
    const long long slot = (long long)(ch.base + (unsigned long long)k);
    if (slot < p.edge_cap) p.edge_pairs[slot] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
  }
}

__device__ __forceinline__ void append_edges(uint64_t mask, int i, int jbase, EdgeChunk& ch,
                                             const ScreenParams& p, int lane) {
  const int cnt = __popcll(mask);
  if (!__any_sync(0xffffffffu, cnt != 0)) return;
  int incl = cnt;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, s);
    if (lane >= s) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (ch.used + total > ch.cap) {
    seal_edges(ch, p, lane);
    const int want = total > SC_EDGE_CHUNK ? total : SC_EDGE_CHUNK;
    unsigned long long nb = 0;
    if (lane == 0) nb = atomicAdd(p.edge_count, (unsigned long long)want);
    ch.base = __shfl_sync(0xffffffffu, nb, 0);
    ch.used = 0;
    ch.cap = want;
  }
  long long slot = (long long)(ch.base + (unsigned long long)(ch.used + incl - cnt));
  ch.used += total;
  while (mask) {
    const int b = __ffsll((long long)mask) - 1;
    mask &= mask - 1;
    ADG_DCHECK(i < p.n && jbase + b < p.n && i < jbase + b);
    if (slot < p.edge_cap) p.edge_pairs[slot] = make_uint2((uint32_t)i, (uint32_t)(jbase + b));
    ++slot;
  }
}

// HMODE 4: the pairs (i, j) of this group whose squared distance may lie
// within row i's radius (candidate j for query i) or column j's (candidate i
// for query j) are appended to knn_out as {query, candidate, lo, hi}; lo / hi
// bracket the exact squared distance (|o - o*| <= eps sn, the screen's error
// model, taken twice).  Each warp appends into 256-slot chunks it reserves
// with one atomic; slots it leaves unused keep the 0xFF sentinel.
struct KnnChunk {
  unsigned long long base;
  int used, cap;
};
constexpr int SC_KNN_CHUNK = 256;

template <bool EDGE, int NP>
__device__ __forceinline__ void epi_knn(const uint32_t* g, const float4* __restrict__ cmeta,
                                        const EpiRow& R, int jbase, int n, float eps2,
                                        KnnChunk& ch, const ScreenParams& p, int lane) {
  uint32_t rmask = 0, cmask = 0;
#pragma unroll
  for (int jj = 0; jj < NP; ++jj) {
    const float4 cm = cmeta[jj];
    const float sn = R.rn + cm.x;
    const float o = fmaf(R.ra2 * cm.z, __uint_as_float(g[jj]), sn);
    const float lo = fmaf(-eps2, sn, o);
    bool rq = lo <= R.rm, cq = lo <= cm.y;
    if (EDGE) {
      const int j = jbase + jj;
      const bool valid = (j > R.i) && (j < n) && (R.i < n);
      rq = rq && valid;
      cq = cq && valid;
    }
    if (rq) rmask |= 1u << jj;
    if (cq) cmask |= 1u << jj;
  }
  const int cnt = __popc(rmask) + __popc(cmask);
  if (!__any_sync(0xffffffffu, cnt != 0)) return;
  int incl = cnt;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, s);
    if (lane >= s) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (ch.used + total > ch.cap) {
    const int want = total > SC_KNN_CHUNK ? total : SC_KNN_CHUNK;
    unsigned long long nb = 0;
    if (lane == 0) nb = atomicAdd(p.near_count, (unsigned long long)want);
    ch.base = __shfl_sync(0xffffffffu, nb, 0);
    ch.used = 0;
    ch.cap = want;
  }
  long long slot = (long long)(ch.base + (unsigned long long)(ch.used + incl - cnt));
  ch.used += total;
  const uint32_t both = rmask | cmask;
#pragma unroll
  for (int jj = 0; jj < NP; ++jj) {
    if ((both >> jj) & 1u) {
      const float4 cm = cmeta[jj];
      const float sn = R.rn + cm.x;
      const float o = fmaf(R.ra2 * cm.z, __uint_as_float(g[jj]), sn);
      const float lo = fmaf(-eps2, sn, o), hi = fmaf(eps2, sn, o);
      const uint32_t j = (uint32_t)(jbase + jj);
      if ((rmask >> jj) & 1u) {
        if (slot < p.near_cap)
          p.knn_out[slot] = make_uint4((uint32_t)R.i, j, __float_as_uint(lo), __float_as_uint(hi));
        ++slot;
      }
      if ((cmask >> jj) & 1u) {
        if (slot < p.near_cap)
          p.knn_out[slot] = make_uint4(j, (uint32_t)R.i, __float_as_uint(lo), __float_as_uint(hi));
        ++slot;
      }
    }
  }
}

// ------------------------------------------------------------- the kernel
// MC (4-CTA clusters, two CTA pairs): the pairs screen two tiles of the same
// 256-row block (p.tiles holds tile pairs: entry 2 t + pair, 0xFFFFFFFF for a
// pair with nothing to do) and share its A rows -- the hi boxes are issued by
// pair 0 and the lo boxes by pair 1, each multicast to the matching CTA of
// both pairs -- so each SM issues half the A requests.  A stage is free once
// both pairs' MMAs committed it (empty barriers count 2).
constexpr uint32_t SC_DUMMY = 0xFFFFFFFFu;

template <int STAGES, int HMODE, bool EDGES, bool MC>
__device__ __forceinline__ void screen_body(const CUtensorMap& map_a_hi, const CUtensorMap& map_a_lo,
                                            const CUtensorMap& map_b_hi, const CUtensorMap& map_b_lo,
                                            const ScreenParams& p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // Carve by byte offsets from the __shared__ array so every access below
  // compiles to LDS/STS; the ring is 1024-aligned (same offset in both CTAs).
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* ring = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + STAGES * SC_STAGE_BYTES);
  uint64_t* full = bars;                // [STAGES]  (used in the leader)
  uint64_t* empty = bars + STAGES;      // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2]       (used in the leader)
  uint64_t* eempty = tempty + 2;        // [1] embedding accumulator read (used in the leader)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(eempty + 2);
  float4* colmeta = reinterpret_cast<float4*>(tmem_slot + 4);          // [2][128]
  double* wsum = reinterpret_cast<double*>(colmeta + 2 * SC_BN);       // [2][16] warp sums
  // histogram counters: bins + 1 real slots (overflow last) and a trash slot
  // for pairs not binned from their screened value
  const int nslot = p.bins + 2;
  unsigned* h32 = reinterpret_cast<unsigned*>(wsum + 2 * SC_EPI_WARPS);  // [nslot] per CTA
  uint8_t* h8 = reinterpret_cast<uint8_t*>(h32 + ((p.bins + 5) & ~3));  // [nslot][512] (HMODE 1)
  unsigned* hw = reinterpret_cast<unsigned*>(h8);                         // [16][nslot] (HMODE 3)
  if (HMODE == 0 && p.hist_scratch) h32 = p.hist_scratch + (size_t)blockIdx.x * nslot;  // large bins

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1u;             // CTA within its pair
  const uint32_t pr = MC ? (crank >> 1) : 0u;   // pair within the cluster
  const uint32_t lead = crank & ~1u;            // cluster rank of the pair's leader
  const bool leader = rank == 0;
  const int64_t cluster = blockIdx.x >> (MC ? 2 : 1);
  const int64_t nclusters = gridDim.x >> (MC ? 2 : 1);
  const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pr));
  const uint16_t empty_mask = MC ? (uint16_t)0xF : (uint16_t)0x3;
  const uint16_t a_mask = (uint16_t)((1u << rank) | (1u << (2 + rank)));  // MC: this CTA's A twins
  auto entry = [&](int64_t t) -> uint32_t { return MC ? p.tiles[2 * t + pr] : p.tiles[t]; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), MC ? 2 : 1);  // MC: both pairs' MMAs release a stage
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), 2 * SC_EPI_WARPS);
    }
    mbar_init(smem_u32(&eempty[0]), 2 * SC_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (warp >= 2) {
    const int et = threadIdx.x - 64;
    for (int b = et; b < nslot; b += SC_EPI_THREADS) h32[b] = 0;
    if (HMODE == 1)
      for (int b = 0; b < nslot; ++b) h8[b * SC_EPI_THREADS + et] = 0;
    if (HMODE == 3)
      for (int b = et; b < SC_EPI_WARPS * nslot; b += SC_EPI_THREADS) hw[b] = 0;
  }
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // one pass over the original K chunks when their lo planes are all zero (the
  // flag is read once, after the stream-ordered prep, by both roles of both CTAs)
  const bool orig1 = p.lo_flag != nullptr && ld_volatile_s32(p.lo_flag) == 0;
  if (warp == 0) {
    // ======================= TMA producer (both CTAs) ============
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a_hi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a_lo)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b_hi)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b_lo)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      int64_t ltp = 0;
      for (int64_t t = p.tile_begin + cluster; t < p.tile_end; t += nclusters, ++ltp) {
        const uint32_t tij = entry(t);
        const bool dummy = MC && tij == SC_DUMMY;
        // MC: the A rows are the pair's block even when this pair has no tile
        const uint32_t tia = dummy ? p.tiles[2 * t + (pr ^ 1u)] : tij;
        const int I2 = (int)(tia >> 16), J = (int)(tij & 0xFFFF);
        const int arow = (p.debug == 6 ? 0 : I2 * SC_PM) + (int)rank * SC_BM;  // 6: A always block 0
        const int brow = J * SC_BN + (int)rank * SC_BNH;
        for (int kc = 0; kc < p.kc_total; ++kc) {
          const uint32_t eb = smem_u32(&empty[stage]);
          while (!mbar_try_wait(eb, phase ^ 1)) __nanosleep(32);  // (hang: see the MMA side's check)
          const uint32_t fb = smem_u32(&full[stage]);
          if constexpr (MC) {
            const uint32_t sbase = smem_u32(ring + stage * SC_STAGE_BYTES);
            // A: pair 0 issues the first slot (hi; or chunk kc in one-pass
            // mode), pair 1 the second (lo; or chunk kc + 1), to both pairs
            const bool one = orig1 && kc < p.kc_orig;
            const bool two = !one || kc + 1 < p.kc_orig;  // second slot in use
            const int nb = (two ? 2 : 1) * (dummy ? 0 : 1);  // B boxes per CTA
            if (leader) mbar_expect_tx(fb, 2 * ((two ? 2 : 1) * SC_A_BYTES + nb * SC_B_BYTES));
            const CUtensorMap* amap = (one || pr == 0) ? &map_a_hi : &map_a_lo;
            const int akc = (one && pr == 1) ? kc + 1 : kc;
            if (pr == 0 || two)
              tma_load_2d_2sm_mc(sbase + pr * SC_A_BYTES, amap, fb, akc * SC_BK, arow, a_mask);
            if (!dummy) {
              tma_load_2d_2sm(sbase + 2 * SC_A_BYTES, &map_b_hi, fb, kc * SC_BK, brow);
              if (two)
                tma_load_2d_2sm(sbase + 2 * SC_A_BYTES + SC_B_BYTES, one ? &map_b_hi : &map_b_lo, fb,
                                (one ? kc + 1 : kc) * SC_BK, brow);
            }
            if (one && two) ++kc;
          } else if (orig1 && kc < p.kc_orig) {
            // hi planes only, two K chunks per stage (the lo slots carry chunk
            // kc + 1): twice the original-side bytes in flight per ring
            const bool two = kc + 1 < p.kc_orig;
            if (leader) mbar_expect_tx(fb, (two ? 4 : 2) * (SC_A_BYTES + SC_B_BYTES));  // both CTAs
            const uint32_t sbase = smem_u32(ring + stage * SC_STAGE_BYTES);
            tma_load_2d_2sm(sbase, &map_a_hi, fb, kc * SC_BK, arow);
            tma_load_2d_2sm(sbase + 2 * SC_A_BYTES, &map_b_hi, fb, kc * SC_BK, brow);
            if (two) {
              tma_load_2d_2sm(sbase + SC_A_BYTES, &map_a_hi, fb, (kc + 1) * SC_BK, arow);
              tma_load_2d_2sm(sbase + 2 * SC_A_BYTES + SC_B_BYTES, &map_b_hi, fb, (kc + 1) * SC_BK, brow);
              ++kc;
            }
          } else if (p.debug == 4) {  // profiling: no loads, just flip the barrier
            if (leader) mbar_arrive_local(fb);
          } else if (p.debug == 5 && (ltp & 1)) {  // profiling: A every other tile only
            if (leader) mbar_expect_tx(fb, 2 * 2 * SC_B_BYTES);
            const uint32_t sbase = smem_u32(ring + stage * SC_STAGE_BYTES);
            tma_load_2d_2sm(sbase + 2 * SC_A_BYTES, &map_b_hi, fb, kc * SC_BK, brow);
            tma_load_2d_2sm(sbase + 2 * SC_A_BYTES + SC_B_BYTES, &map_b_lo, fb, kc * SC_BK, brow);
          } else {
            if (leader) mbar_expect_tx(fb, 2 * SC_STAGE_BYTES);  // both CTAs' bytes
            const uint32_t sbase = smem_u32(ring + stage * SC_STAGE_BYTES);
            tma_load_2d_2sm(sbase, &map_a_hi, fb, kc * SC_BK, arow);
            tma_load_2d_2sm(sbase + SC_A_BYTES, &map_a_lo, fb, kc * SC_BK, arow);
            tma_load_2d_2sm(sbase + 2 * SC_A_BYTES, &map_b_hi, fb, kc * SC_BK, brow);
            tma_load_2d_2sm(sbase + 2 * SC_A_BYTES + SC_B_BYTES, &map_b_lo, fb, kc * SC_BK, brow);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader CTA) ============
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int64_t lt = 0;
      const bool skip_mma = p.debug == 2 || p.debug == 3;
      for (int64_t t = p.tile_begin + cluster; t < p.tile_end; t += nclusters) {
        if (MC && entry(t) == SC_DUMMY) {
          // no tile for this pair: consume the stages (the other pair needs
          // their A boxes) without MMAs
          for (int kc = 0; kc < p.kc_total; ++kc) {
            mbar_wait(smem_u32(&full[stage]), phase);
            tc_fence_after();
            if (orig1 && kc < p.kc_orig && kc + 1 < p.kc_orig) ++kc;
            tc_commit_mask(smem_u32(&empty[stage]), empty_mask);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          continue;
        }
        const int b = (int)(lt & 1);
        const uint32_t use = (uint32_t)(lt >> 1);
        mbar_wait(smem_u32(&tempty[b]), (use & 1) ^ 1);
        tc_fence_after();
        // TMEM: orig accumulators double-buffered at [0,160) / [160,320); the
        // embedding accumulator (last K chunk of a tile) single-buffered at
        // [320,480): the epilogue reads it ~a tile's orig MMAs before it is
        // needed again
        const uint32_t d_orig = tmem_base + (uint32_t)(b * SC_BN);
        const uint32_t d_emb = tmem_base + (uint32_t)(2 * SC_BN);
        for (int kc = 0; kc < p.kc_total; ++kc) {
          mbar_wait(smem_u32(&full[stage]), phase);
          if (kc == p.kc_orig) mbar_wait(smem_u32(&eempty[0]), ((uint32_t)lt & 1) ^ 1);
          tc_fence_after();
          const bool is_emb = kc >= p.kc_orig;
          const uint32_t dacc = is_emb ? d_emb : d_orig;
          const bool first = (kc == 0) || (kc == p.kc_orig);
          const int nk = skip_mma ? 0
                         : (kc == p.kc_orig - 1)  ? p.k16_last_orig
                         : (kc == p.kc_total - 1) ? p.k16_last_emb
                                                  : SC_K16;
          // descriptors differ only in the start-address field (addr >> 4, no
          // carry out of its 14 bits below 256 KB): one base + constant offsets
          const uint64_t d0 = sw128_desc(smem_u32(ring + stage * SC_STAGE_BYTES));
          constexpr uint64_t OA_LO = SC_A_BYTES >> 4, OB_HI = (2 * SC_A_BYTES) >> 4,
                             OB_LO = (2 * SC_A_BYTES + SC_B_BYTES) >> 4;
          if (orig1 && !is_emb) {
            // chunk kc from the hi slots, chunk kc + 1 (if any) from the lo slots
#pragma unroll
            for (int k = 0; k < SC_K16; ++k) {
              if (k < nk) {
                const uint64_t kd = d0 + (uint64_t)(2 * k);
                tc_mma_f16_pair(dacc, kd, kd + OB_HI, SC_IDESC, (first && k == 0) ? 0u : 1u);
              }
            }
            if (kc + 1 < p.kc_orig) {
              ++kc;
              const int nk2 = skip_mma ? 0 : (kc == p.kc_orig - 1) ? p.k16_last_orig : SC_K16;
#pragma unroll
              for (int k = 0; k < SC_K16; ++k) {
                if (k < nk2) {
                  const uint64_t kd = d0 + (uint64_t)(2 * k);
                  tc_mma_f16_pair(dacc, kd + OA_LO, kd + OB_LO, SC_IDESC, 1u);
                }
              }
            }
          } else {
#pragma unroll
            for (int k = 0; k < SC_K16; ++k) {
              if (k < nk) {
                const uint64_t kd = d0 + (uint64_t)(2 * k);  // 16 fp16 = 32 bytes along K
                tc_mma3_f16_pair(dacc, kd, kd + OA_LO, kd + OB_HI, kd + OB_LO,
                                 (first && k == 0) ? 0u : 1u);
              }
            }
          }
          tc_commit_mask(smem_u32(&empty[stage]), empty_mask);  // frees the slot (MC: in all four CTAs)
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit_mask(smem_u32(&tfull[b]), pair_mask);  // this tile's accumulators are ready (the pair)
        ++lt;
      }
    }
  } else {
    // ======================= epilogue (warps 2..17) =============
    const int et = threadIdx.x - 64;                        // 0..511
    const int quarter = warp & 3;                           // TMEM lane quarter of this warp
    const int cslot = (warp - 2) >> 2;                      // 32-column slot of the tile
    const int col0 = cslot * SC_COLS_PER_WARP;
    const int row_in_tile = quarter * 32 + lane;
    uint8_t* hrow = h8 + et;                                // private u8 counters (stride 512)
    unsigned* hcnt = HMODE == 3 ? hw + (warp - 2) * nslot : h32;  // this warp's counters
    const int bins = p.bins;
    const float tau = p.tau, eps = p.eps;
    const float hbias = p.hist_scale;
    const float hcap = 8388608.0f + (float)bins;
    const float ef = p.edge_f;
    int64_t lt = 0;
    KnnChunk kch{0ull, 0, 0};  // HMODE 4: this warp's current append chunk
    EdgeChunk ech{0ull, 0, 0};  // this warp's current edge-list chunk
    int64_t prev_slot = 0;  // canonical slot of the previous tile: the partial sums'
                            // order then does not depend on the order tiles are visited in
    // the next tile's list entry, slot and this thread's column metadata are
    // fetched a tile ahead, so the per-tile barrier never waits on global loads
    uint32_t tij_n = 0;
    int64_t slot_n = 0;
    float4 cm_n = make_float4(0.f, 0.f, 0.f, 0.f);
    auto prefetch = [&](int64_t tt) {
      if (tt < p.tile_end) {
        tij_n = entry(tt);
        slot_n = p.tile_slots[MC ? 2 * tt + pr : tt];
        if (et < SC_BN && !(MC && tij_n == SC_DUMMY)) {
          const int64_t c = (int64_t)(tij_n & 0xFFFF) * SC_BN + et;
          cm_n = p.meta[c];
          if (HMODE == 4) cm_n.y = p.row_tau2[c];
        }
      }
    };
    prefetch(p.tile_begin + cluster);
    for (int64_t t = p.tile_begin + cluster; t < p.tile_end; t += nclusters) {
      const int b = (int)(lt & 1);
      const uint32_t use = (uint32_t)(lt >> 1);
      const uint32_t tij = tij_n;
      const int I2 = (int)(tij >> 16), J = (int)(tij & 0xFFFF);
      const int64_t slot = slot_n;
      if (MC && tij == SC_DUMMY) {  // no tile for this pair (uniform over the epilogue warps)
        prefetch(t + nclusters);
        continue;
      }
      if (et < SC_BN) colmeta[b * SC_BN + et] = cm_n;
      prefetch(t + nclusters);
      asm volatile("bar.sync 1, %0;" ::"n"(SC_EPI_THREADS) : "memory");
      if (HMODE != 2 && HMODE != 4 && lt > 0 && (lt % SC_GFLUSH_TILES) == 0) {
        // per-CTA / per-warp u32 counts -> global u64 long before they could wrap
        for (int bb = et; bb <= bins; bb += SC_EPI_THREADS)
          if (h32[bb]) {
            atomicAdd(&p.hist[bb], (unsigned long long)h32[bb]);
            h32[bb] = 0;
          }
        if (HMODE == 3)
          for (int q = et; q < SC_EPI_WARPS * nslot; q += SC_EPI_THREADS)
            if (q % nslot <= bins && hw[q]) {
              atomicAdd(&p.hist[q % nslot], (unsigned long long)hw[q]);
              hw[q] = 0;
            }
        asm volatile("bar.sync 1, %0;" ::"n"(SC_EPI_THREADS) : "memory");
      }
      if (HMODE != 4 && et == 0 && lt > 0) {
        // previous tile's 16 warp sums are in smem (written before this
        // barrier): one slot per CTA per tile, summed in fixed warp order
        double s = 0.0;
        for (int w = 0; w < SC_EPI_WARPS; ++w) s += wsum[(b ^ 1) * SC_EPI_WARPS + w];
        p.tile_sums[prev_slot * 2 + rank] = s;
      }
      prev_slot = slot;
      const int row0 = I2 * SC_PM + (int)rank * SC_BM;
      EpiRow R;
      R.i = row0 + row_in_tile;
      {
        const float4 rmeta = p.meta[R.i];
        R.rn = rmeta.x;
        R.rm = HMODE == 4 ? p.row_tau2[R.i] : rmeta.y;
        R.ra2 = -2.0f * rmeta.z;
        R.rb2 = -2.0f * rmeta.w;
      }
      R.vmax = 0.0f;
      R.umax = 0.0f;
      // tiles touching the diagonal or the padding need the validity mask
      const bool edge = (J * SC_BN < row0 + SC_BM) || ((J + 1) * SC_BN > p.n) || (row0 + SC_BM > p.n);
      mbar_wait(smem_u32(&tfull[b]), use & 1);
      tc_fence_after();
      const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
      const uint32_t ta_orig = tmem_base + lane_off + (uint32_t)(b * SC_BN + col0);
      const uint32_t ta_emb = tmem_base + lane_off + (uint32_t)(2 * SC_BN + col0);
      float tsum = 0.0f;
      uint64_t edgem = 0, nearm = 0;  // this row's edge / near-coincident pairs (bit = column)
      uint64_t excl = 0;              // !EDGES: pairs binned as 0 that do not count
      const float4* cmeta = colmeta + b * SC_BN + col0;
      const int jbase = J * SC_BN + col0;
      // the warp's 40 columns as 16 + 16 + 8 (32 accumulator registers live)
#pragma unroll 1
      for (int grp = 0; grp < 3; ++grp) {
        const int c = grp * 16;
        uint32_t g[16], h[16];
        if (grp < 2) {
          TMEM_LD16(ta_orig + (uint32_t)c, g);
          if (HMODE != 4) TMEM_LD16(ta_emb + (uint32_t)c, h);
        } else {
          TMEM_LD8(ta_orig + (uint32_t)c, g);
          if (HMODE != 4) TMEM_LD8(ta_emb + (uint32_t)c, h);
        }
        tmem_ld_wait();
        if (grp == 2) {
          // all of this warp's columns are in registers: release both buffers
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_cluster(smem_u32(&tempty[b]), lead);
            mbar_arrive_cluster(smem_u32(&eempty[0]), lead);
          }
        }
        if constexpr (HMODE == 4) {
          if (grp < 2) {
            if (edge)
              epi_knn<true, 16>(g, cmeta + c, R, jbase + c, p.n, 2.0f * eps, kch, p, lane);
            else
              epi_knn<false, 16>(g, cmeta + c, R, jbase + c, p.n, 2.0f * eps, kch, p, lane);
          } else {
            if (edge)
              epi_knn<true, 8>(g, cmeta + c, R, jbase + c, p.n, 2.0f * eps, kch, p, lane);
            else
              epi_knn<false, 8>(g, cmeta + c, R, jbase + c, p.n, 2.0f * eps, kch, p, lane);
          }
        } else if (p.debug == 1 || p.debug >= 3) {
          tsum += __uint_as_float(g[0] ^ g[7] ^ h[3] ^ h[5]);  // keep the loads live
        } else if (grp < 2) {
          if (edge)
            epi_pairs<true, HMODE, 16, EDGES>(g, h, cmeta + c, hrow, hcnt, R, tsum, jbase + c, p.n, tau, eps,
                                       hbias, hcap, ef, edgem, nearm, excl, c);
          else
            epi_pairs<false, HMODE, 16, EDGES>(g, h, cmeta + c, hrow, hcnt, R, tsum, jbase + c, p.n, tau, eps,
                                        hbias, hcap, ef, edgem, nearm, excl, c);
        } else {
          if (edge)
            epi_pairs<true, HMODE, 8, EDGES>(g, h, cmeta + c, hrow, hcnt, R, tsum, jbase + c, p.n, tau, eps,
                                      hbias, hcap, ef, edgem, nearm, excl, c);
          else
            epi_pairs<false, HMODE, 8, EDGES>(g, h, cmeta + c, hrow, hcnt, R, tsum, jbase + c, p.n, tau, eps,
                                       hbias, hcap, ef, edgem, nearm, excl, c);
        }
      }
      if constexpr (HMODE == 4) {
        // candidates were appended per group
      } else {
        if constexpr (HMODE != 2 && EDGES) append_edges(edgem, R.i, jbase, ech, p, lane);
        if constexpr (!EDGES) {
          if (excl) {
            if constexpr (HMODE == 1)
              hrow[0] = (uint8_t)(hrow[0] - __popcll(excl));
            else if constexpr (HMODE == 0 || HMODE == 3)
              atomicSub(&hcnt[0], (unsigned)__popcll(excl));
          }
        }
        while (nearm) {
          const int jj = __ffsll((long long)nearm) - 1;
          ADG_DCHECK(R.i < p.n && jbase + jj < p.n && R.i < jbase + jj);
          nearm &= nearm - 1;
          const unsigned long long slot = atomicAdd(p.near_count, 1ull);
          if ((long long)slot < p.near_cap) {
            p.near_pairs[2 * slot] = (uint32_t)R.i;
            p.near_pairs[2 * slot + 1] = (uint32_t)(jbase + jj);
          }
        }
      }
      if (HMODE != 4 && R.i < p.n) {
        if (R.vmax > 0.0f) atomicMax(reinterpret_cast<int*>(p.row_max) + R.i, __float_as_int(R.vmax));
        if (R.umax > 0.0f) atomicMax(reinterpret_cast<int*>(p.row_bound) + R.i, __float_as_int(R.umax));
      }
      // warp sum in fp32 (fixed shuffle pattern: deterministic), fp64 from there
      float wsum32 = tsum;
#pragma unroll
      for (int s = 16; s; s >>= 1) wsum32 += __shfl_xor_sync(0xffffffffu, wsum32, s);
      if (lane == 0) wsum[b * SC_EPI_WARPS + (warp - 2)] = (double)wsum32;
      if (HMODE == 1 && ((lt + 1) % SC_FLUSH_TILES) == 0) {
        // private u8 counters -> per-CTA u32 histogram before they can wrap:
        // one warp reduction and one atomic per bin (not 32 same-address atomics)
#pragma unroll 4
        for (int bb = 0; bb <= bins; ++bb) {
          const unsigned cnt = hrow[bb * SC_EPI_THREADS];
          const unsigned tot = __reduce_add_sync(0xffffffffu, cnt);
          if (tot) {  // warp-uniform
            if (lane == 0) atomicAdd(&h32[bb], tot);
            hrow[bb * SC_EPI_THREADS] = 0;
          }
        }
      }
      ++lt;
    }
    if (HMODE == 1)
      for (int bb = 0; bb <= bins; ++bb) {
        const unsigned tot = __reduce_add_sync(0xffffffffu, (unsigned)hrow[bb * SC_EPI_THREADS]);
        if (tot && lane == 0) atomicAdd(&h32[bb], tot);
      }
    if (HMODE != 2 && HMODE != 4 && EDGES) seal_edges(ech, p, lane);
    asm volatile("bar.sync 1, %0;" ::"n"(SC_EPI_THREADS) : "memory");
    if (HMODE != 4 && et == 0 && lt > 0) {  // the last tile's sum
      double s = 0.0;
      for (int w = 0; w < SC_EPI_WARPS; ++w) s += wsum[((lt - 1) & 1) * SC_EPI_WARPS + w];
      p.tile_sums[prev_slot * 2 + rank] = s;
    }
    if (HMODE != 2 && HMODE != 4)
      for (int bb = et; bb <= bins; bb += SC_EPI_THREADS)
        if (h32[bb]) atomicAdd(&p.hist[bb], (unsigned long long)h32[bb]);
    if (HMODE == 3)
      for (int q = et; q < SC_EPI_WARPS * nslot; q += SC_EPI_THREADS)
        if (q % nslot <= bins && hw[q]) atomicAdd(&p.hist[q % nslot], (unsigned long long)hw[q]);
  }

  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base)
                 : "memory");
  }
}

template <int STAGES, int HMODE, bool EDGES = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SC_THREADS, 1)
screen_kernel(const __grid_constant__ CUtensorMap map_a_hi, const __grid_constant__ CUtensorMap map_a_lo,
              const __grid_constant__ CUtensorMap map_b_hi, const __grid_constant__ CUtensorMap map_b_lo,
              const ScreenParams p) {
  screen_body<STAGES, HMODE, EDGES, false>(map_a_hi, map_a_lo, map_b_hi, map_b_lo, p);
}

// two CTA pairs sharing A by multicast (p.tiles: tile pairs, p.tile_begin /
// p.tile_end count pairs)
template <int STAGES, int HMODE, bool EDGES = false>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(SC_THREADS, 1)
screen_mc_kernel(const __grid_constant__ CUtensorMap map_a_hi, const __grid_constant__ CUtensorMap map_a_lo,
                 const __grid_constant__ CUtensorMap map_b_hi, const __grid_constant__ CUtensorMap map_b_lo,
                 const ScreenParams p) {
  screen_body<STAGES, HMODE, EDGES, true>(map_a_hi, map_a_lo, map_b_hi, map_b_lo, p);
}

}  // namespace adg
