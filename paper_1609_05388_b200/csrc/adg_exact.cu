// adg_exact.cu -- exact fp64 distortion kernels (sm_100a, SIMT fp64).
//
// The reference's own per-pair formula (proj/src/distortion.cpp:59-75):
// direct differences in fp64, a pair is "zero" iff its fp64 orig_sq == 0.0,
// value = |sqrt(emb_sq)/sqrt(orig_sq) - 1|, binned by distortion.cpp:81-87.
// Used (a) as the EXACT engine for small jobs and the sampled mode, with the
// reference's block structure (16384-pair blocks, Neumaier inside, ordered
// merge, distortion.cpp:139-190) so results do not depend on GPU count; and
// (b) as the refine step of the SCREEN engine (candidate rows, near-zero
// pairs).
#include "adg_exact.cuh"

#include <type_traits>

namespace adg {

constexpr int EX_THREADS = 256;
constexpr uint64_t EX_BLOCK = 16384;  // distortion.hpp:54 default, fixed here
constexpr int EX_PER_THREAD = (int)(EX_BLOCK / EX_THREADS);

// proj/src/distortion.cpp:46-57
__device__ void decode_pair_dev(uint64_t p, uint64_t n, uint64_t& i, uint64_t& j) {
  const double nn = (double)n;
  double guess = floor((2.0 * nn - 1.0 - sqrt((2.0 * nn - 1.0) * (2.0 * nn - 1.0) - 8.0 * (double)p)) / 2.0);
  if (guess < 0.0) guess = 0.0;
  i = (uint64_t)guess;
  auto row_start = [n](uint64_t r) { return r * (2 * n - r - 1) / 2; };
  while (i > 0 && row_start(i) > p) --i;
  while (row_start(i + 1) <= p) ++i;
  j = i + 1 + (p - row_start(i));
}

// proj/src/distortion.cpp:59-75 for one pair; returns -1 for a zero pair.
template <typename TO, typename TE>
__device__ __forceinline__ double pair_value_dev(const TO* __restrict__ X, int64_t d,
                                                 const TE* __restrict__ Y, int64_t r, uint64_t i,
                                                 uint64_t j) {
  const TO* xi = X + i * d;
  const TO* xj = X + j * d;
  double o = 0.0;
  for (int64_t t = 0; t < d; ++t) {
    const double df = to_f64(xi[t]) - to_f64(xj[t]);
    o = fma(df, df, o);
  }
  if (o == 0.0) return -1.0;
  const TE* fi = Y + i * r;
  const TE* fj = Y + j * r;
  double e = 0.0;
  for (int64_t t = 0; t < r; ++t) {
    const double df = to_f64(fi[t]) - to_f64(fj[t]);
    e = fma(df, df, e);
  }
  return fabs(sqrt(e) / sqrt(o) - 1.0);
}

__device__ __forceinline__ void neumaier_add(double& sum, double& comp, double v) {
  const double t = sum + v;
  if (fabs(sum) >= fabs(v))
    comp += (sum - t) + v;
  else
    comp += (v - t) + sum;
  sum = t;
}

__device__ __forceinline__ int bin_of(double value, int bins, double hist_max) {
  // proj/src/distortion.cpp:81-87
  if (value >= hist_max) return bins;
  uint64_t b = (uint64_t)(value / hist_max * bins);
  if (b > (uint64_t)(bins - 1)) b = (uint64_t)(bins - 1);
  return (int)b;
}

// One CTA per 16384-pair block; each thread owns 64 consecutive pairs.
template <typename TO, typename TE>
__global__ void __launch_bounds__(EX_THREADS)
exact_block_kernel(const TO* __restrict__ X, int64_t n, int64_t d, const TE* __restrict__ Y,
                   int64_t r, const uint64_t* __restrict__ sampled, uint64_t work, int bins,
                   double hist_max, BlockOut* __restrict__ out, unsigned long long* __restrict__ hist,
                   bool global_hist) {
  extern __shared__ unsigned int sh_hist[];
  __shared__ double s_sum[EX_THREADS], s_comp[EX_THREADS], s_max[EX_THREADS];
  __shared__ uint64_t s_arg[EX_THREADS], s_ev[EX_THREADS], s_zero[EX_THREADS];
  if (!global_hist)
    for (int b = threadIdx.x; b <= bins; b += EX_THREADS) sh_hist[b] = 0;
  __syncthreads();
  const uint64_t block = blockIdx.x;
  const uint64_t begin = block * EX_BLOCK + (uint64_t)threadIdx.x * EX_PER_THREAD;
  uint64_t end = begin + EX_PER_THREAD;
  if (end > work) end = work;
  const uint64_t bend = (block + 1) * EX_BLOCK < work ? (block + 1) * EX_BLOCK : work;
  if (end > bend) end = bend;
  double sum = 0.0, comp = 0.0, mx = -1.0;
  uint64_t arg = UINT64_MAX, ev = 0, zero = 0;
  uint64_t i = 0, j = 0;
  if (!sampled && begin < end) decode_pair_dev(begin, (uint64_t)n, i, j);
  for (uint64_t p = begin; p < end; ++p) {
    uint64_t pid = p;
    if (sampled) {
      pid = sampled[p];
      decode_pair_dev(pid, (uint64_t)n, i, j);
    } else if (p != begin) {
      if (++j >= (uint64_t)n) {
        ++i;
        j = i + 1;
      }
    }
    const double v = pair_value_dev(X, d, Y, r, i, j);
    if (v < 0.0) {
      ++zero;
      continue;
    }
    if (v > mx) {
      mx = v;
      arg = pid;
    }
    neumaier_add(sum, comp, v);
    ++ev;
    if (global_hist)
      atomicAdd(&hist[bin_of(v, bins, hist_max)], 1ull);
    else
      atomicAdd(&sh_hist[bin_of(v, bins, hist_max)], 1u);
  }
  s_sum[threadIdx.x] = sum;
  s_comp[threadIdx.x] = comp;
  s_max[threadIdx.x] = mx;
  s_arg[threadIdx.x] = arg;
  s_ev[threadIdx.x] = ev;
  s_zero[threadIdx.x] = zero;
  __syncthreads();
  if (threadIdx.x == 0) {
    // Fixed thread order => deterministic block totals.
    double bs = 0.0, bc = 0.0, bm = -1.0;
    uint64_t ba = UINT64_MAX, be = 0, bz = 0;
    for (int t = 0; t < EX_THREADS; ++t) {
      neumaier_add(bs, bc, s_sum[t] + s_comp[t]);
      if (s_max[t] > bm) {
        bm = s_max[t];
        ba = s_arg[t];
      }
      be += s_ev[t];
      bz += s_zero[t];
    }
    out[block] = BlockOut{bs + bc, bm, ba, be, bz};
  }
  if (!global_hist)
    for (int b = threadIdx.x; b <= bins; b += EX_THREADS)
      if (sh_hist[b]) atomicAdd(&hist[b], (unsigned long long)sh_hist[b]);
}

// Ordered merge of block results (distortion.cpp:178-190).
__global__ void merge_blocks_kernel(const BlockOut* __restrict__ blocks, uint64_t nblocks,
                                    MergeOut* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0, c = 0.0, mx = -1.0;
  uint64_t arg = UINT64_MAX, ev = 0, zero = 0;
  for (uint64_t b = 0; b < nblocks; ++b) {
    const BlockOut& o = blocks[b];
    neumaier_add(s, c, o.sum);
    if (o.max > mx) {
      mx = o.max;
      arg = o.argp;
    }
    ev += o.evaluated;
    zero += o.zero;
  }
  out->sum = s + c;
  out->max = mx;
  out->argp = arg;
  out->evaluated = ev;
  out->zero = zero;
}

template <typename TO, typename TE>
static void run_exact_typed(adg_ctx* ctx, const TO* X, int64_t n, int64_t d, const TE* Y, int64_t r,
                            const uint64_t* sampled, uint64_t work, int bins, double hist_max,
                            unsigned long long* hist_dev, MergeOut* merged_dev) {
  const uint64_t nblocks = work == 0 ? 0 : (work + EX_BLOCK - 1) / EX_BLOCK;
  DevBuf<BlockOut> blocks(nblocks ? nblocks : 1, ctx->stream);
  if (nblocks) {
    // per-CTA u32 counters in shared memory (beside the kernel's 12 KB of
    // static reduction arrays) up to 160 KB of bins, else u64 atomics on the
    // global histogram (any bin count; integer adds, so still deterministic)
    const size_t sh = (size_t)(bins + 1) * sizeof(unsigned);
    const bool global_hist = sh > 160 * 1024;
    auto kern = exact_block_kernel<TO, TE>;
    if (!global_hist)
      ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    kern<<<(unsigned)nblocks, EX_THREADS, global_hist ? 0 : sh, ctx->stream>>>(
        X, n, d, Y, r, sampled, work, bins, hist_max, blocks.ptr, hist_dev, global_hist);
    after_launch(ctx);
  }
  merge_blocks_kernel<<<1, 32, 0, ctx->stream>>>(blocks.ptr, nblocks, merged_dev);
  after_launch(ctx);
}

void run_exact(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d, const void* Y,
               adg_dtype yd, int64_t r, const uint64_t* sampled, uint64_t work, int bins,
               double hist_max, unsigned long long* hist_dev, MergeOut* merged_dev) {
  ADG_REQUIRE(yd == ADG_F64 || yd == ADG_F32 || yd == ADG_BF16, "evaluate: bad embedded dtype");
  ADG_DISPATCH_DTYPE(xd, TO, {
    ADG_DISPATCH_DTYPE(yd, TE, {
      run_exact_typed<TO, TE>(ctx, (const TO*)X, n, d, (const TE*)Y, r, sampled, work, bins,
                              hist_max, hist_dev, merged_dev);
    });
  });
}

// ------------------------------------------------------ candidate rows
// For each listed row i, every pair (i, j > i): exact value, max and the
// lowest j attaining it.  One CTA per (row, j-chunk); each warp takes JW j's
// at a time with lanes over coordinates, 16-byte loads when rows are 16-byte
// aligned (a warp reads 512 contiguous bytes of a row per load, JW rows in
// flight), x_i staged in smem as fp64.  Streaming-bound: one row reads all
// of X's later rows once.
constexpr int RR_THREADS = 256;
// j's per CTA: n / 444 (at least 64), so one refined row is ~444 CTAs -- three
// resident per SM on a 148-SM B200 (80 registers), one balanced wave (C3:
// 79 -> 49 us against 64-row chunks in ~3 waves).  A function of n only: every
// rank of a sharded refine splits the same chunks.
constexpr int64_t RR_TARGET_CTAS = 444;
static int64_t rr_chunk(int64_t n) {
  return std::max<int64_t>(64, (n + RR_TARGET_CTAS - 1) / RR_TARGET_CTAS);
}

int64_t row_refine_chunks(int64_t n) { return n / rr_chunk(n) + 1; }

template <typename TO, typename TE, bool VEC>
__global__ void __launch_bounds__(RR_THREADS, 3)
row_refine_kernel(const TO* __restrict__ X, int64_t n, int64_t d, const TE* __restrict__ Y,
                  int64_t r, const int64_t* __restrict__ rows, RowBest* __restrict__ out,
                  int64_t chunks_per_row, int64_t chunk0, int64_t chunk_rows) {
  // blocks: rows x chunks_per_row chunks, the row's chunks [chunk0, chunk0 + chunks_per_row)
  extern __shared__ double sh[];
  double* xi = sh;       // d
  double* fi = sh + d;   // r
  __shared__ double w_max[RR_THREADS / 32];
  __shared__ int64_t w_arg[RR_THREADS / 32];
  const int64_t row_slot = blockIdx.x / chunks_per_row;
  const int64_t chunk = chunk0 + blockIdx.x % chunks_per_row;
  const int64_t i = rows[row_slot];
  if (i < 0) {  // no row selected (nothing screened above zero)
    if (threadIdx.x == 0) out[blockIdx.x] = RowBest{-1.0, -1, -1};
    return;
  }
  for (int64_t t = threadIdx.x; t < d; t += RR_THREADS) xi[t] = to_f64(X[i * d + t]);
  for (int64_t t = threadIdx.x; t < r; t += RR_THREADS) fi[t] = to_f64(Y[i * r + t]);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j0 = i + 1 + chunk * chunk_rows;
  int64_t j1 = j0 + chunk_rows;
  if (j1 > n) j1 = n;
  double best = -1.0;
  int64_t barg = INT64_MAX;
  constexpr int JW = 4;  // j's per warp iteration (x 4 unrolled K steps: 16 loads in flight)
  for (int64_t jb = j0 + warp * JW; jb < j1; jb += (RR_THREADS / 32) * JW) {
    double o[JW], e[JW];
#pragma unroll
    for (int q = 0; q < JW; ++q) o[q] = e[q] = 0.0;
    if constexpr (VEC && std::is_same<TO, float>::value) {
#pragma unroll 4
      for (int64_t t = 4 * lane; t < d; t += 128) {
        const double x0 = xi[t], x1 = xi[t + 1], x2 = xi[t + 2], x3 = xi[t + 3];
        float4 v[JW];
#pragma unroll
        for (int q = 0; q < JW; ++q)
          v[q] = (jb + q < j1) ? __ldcs(reinterpret_cast<const float4*>(X + (jb + q) * d + t))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < JW; ++q) {
          double df = x0 - (double)v[q].x;
          o[q] = fma(df, df, o[q]);
          df = x1 - (double)v[q].y;
          o[q] = fma(df, df, o[q]);
          df = x2 - (double)v[q].z;
          o[q] = fma(df, df, o[q]);
          df = x3 - (double)v[q].w;
          o[q] = fma(df, df, o[q]);
        }
      }
    } else {
      for (int64_t t = lane; t < d; t += 32) {
        const double xv = xi[t];
#pragma unroll
        for (int q = 0; q < JW; ++q)
          if (jb + q < j1) {
            const double df = xv - to_f64(X[(jb + q) * d + t]);
            o[q] = fma(df, df, o[q]);
          }
      }
    }
    for (int64_t t = lane; t < r; t += 32) {
      const double fv = fi[t];
#pragma unroll
      for (int q = 0; q < JW; ++q)
        if (jb + q < j1) {
          const double df = fv - to_f64(Y[(jb + q) * r + t]);
          e[q] = fma(df, df, e[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < JW; ++q)
      for (int s = 16; s; s >>= 1) {
        o[q] += __shfl_xor_sync(0xffffffffu, o[q], s);
        e[q] += __shfl_xor_sync(0xffffffffu, e[q], s);
      }
#pragma unroll
    for (int q = 0; q < JW; ++q) {
      if (jb + q >= j1 || o[q] == 0.0) continue;  // zero pair: not evaluated (distortion.cpp:66-69)
      const double v = fabs(sqrt(e[q]) / sqrt(o[q]) - 1.0);
      if (v > best) {  // j increases within a warp, so ties keep the lowest j
        best = v;
        barg = jb + q;
      }
    }
  }
  if (lane == 0) {
    w_max[warp] = best;
    w_arg[warp] = barg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bm = -1.0;
    int64_t ba = INT64_MAX;
    for (int w = 0; w < RR_THREADS / 32; ++w)
      if (w_max[w] > bm || (w_max[w] == bm && w_arg[w] < ba)) {
        bm = w_max[w];
        ba = w_arg[w];
      }
    out[blockIdx.x] = RowBest{bm, i, ba};
  }
}

// Many candidate rows (loose screen bounds, e.g. a map that nearly collapses
// many pairs): RB rows per CTA share every X[j] / Y[j] load.  Lane = one j;
// the RB rows sit in smem (broadcast reads), fp64 FMAs per lane per
// coordinate, no shuffles inside the loop.  j increases per lane and warps
// reduce with the lowest-j tie rule, as row_refine_kernel.
constexpr int RB_ROWS = 8, RB_CHUNK = 1024;

template <typename TO, typename TE, bool VEC>
__global__ void __launch_bounds__(RR_THREADS)
row_refine_batch_kernel(const TO* __restrict__ X, int64_t n, int64_t d, const TE* __restrict__ Y,
                        int64_t r, const int64_t* __restrict__ rows, int64_t nrows,
                        RowBest* __restrict__ out, int64_t chunks) {
  extern __shared__ double sh[];
  double* xs = sh;                 // [RB_ROWS][d]
  double* fs = sh + RB_ROWS * d;   // [RB_ROWS][r]
  __shared__ double w_max[RR_THREADS / 32][RB_ROWS];
  __shared__ int64_t w_arg[RR_THREADS / 32][RB_ROWS];
  const int64_t batch = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
  int64_t ri[RB_ROWS];
  int64_t imin = INT64_MAX;
#pragma unroll
  for (int q = 0; q < RB_ROWS; ++q) {
    const int64_t slot = batch * RB_ROWS + q;
    ri[q] = slot < nrows ? rows[slot] : -1;
    if (ri[q] >= 0 && ri[q] < imin) imin = ri[q];
  }
  const int64_t j0 = chunk * RB_CHUNK;
  const int64_t j1 = min(n, j0 + RB_CHUNK);
  const bool active = imin != INT64_MAX && j1 > imin + 1;
  if (active) {
    for (int64_t t = threadIdx.x; t < RB_ROWS * d; t += RR_THREADS) {
      const int64_t q = t / d, c = t % d;
      xs[t] = ri[q] >= 0 ? to_f64(X[ri[q] * d + c]) : 0.0;
    }
    for (int64_t t = threadIdx.x; t < RB_ROWS * r; t += RR_THREADS) {
      const int64_t q = t / r, c = t % r;
      fs[t] = ri[q] >= 0 ? to_f64(Y[ri[q] * r + c]) : 0.0;
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double best[RB_ROWS];
  int64_t barg[RB_ROWS];
#pragma unroll
  for (int q = 0; q < RB_ROWS; ++q) {
    best[q] = -1.0;
    barg[q] = INT64_MAX;
  }
  if (active) {
    for (int64_t jb = max(j0, imin + 1) + threadIdx.x; jb < j1; jb += RR_THREADS) {
      const int64_t j = jb;
      double o[RB_ROWS], e[RB_ROWS];
#pragma unroll
      for (int q = 0; q < RB_ROWS; ++q) o[q] = e[q] = 0.0;
      int64_t t = 0;
      if (VEC) {  // 4 coordinates per load (16 B fp32 / 8 B bf16): 4x fewer L1 wavefronts
        for (; t + 4 <= d; t += 4) {
          double xv[4];
          if constexpr (std::is_same<TO, float>::value) {
            const float4 v4 = __ldg(reinterpret_cast<const float4*>(X + j * d + t));
            xv[0] = v4.x, xv[1] = v4.y, xv[2] = v4.z, xv[3] = v4.w;
          } else if constexpr (std::is_same<TO, __nv_bfloat16>::value) {
            const uint2 u = __ldg(reinterpret_cast<const uint2*>(X + j * d + t));
            xv[0] = __uint_as_float(u.x << 16), xv[1] = __uint_as_float(u.x & 0xffff0000u);
            xv[2] = __uint_as_float(u.y << 16), xv[3] = __uint_as_float(u.y & 0xffff0000u);
          } else {
            const double2 a = __ldg(reinterpret_cast<const double2*>(X + j * d + t));
            const double2 b = __ldg(reinterpret_cast<const double2*>(X + j * d + t + 2));
            xv[0] = a.x, xv[1] = a.y, xv[2] = b.x, xv[3] = b.y;
          }
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int q = 0; q < RB_ROWS; ++q) {
              const double df = xs[q * d + t + c] - xv[c];
              o[q] = fma(df, df, o[q]);
            }
        }
      }
      for (; t < d; ++t) {
        const double xv = to_f64(X[j * d + t]);
#pragma unroll
        for (int q = 0; q < RB_ROWS; ++q) {
          const double df = xs[q * d + t] - xv;
          o[q] = fma(df, df, o[q]);
        }
      }
      for (int64_t t = 0; t < r; ++t) {
        const double fv = to_f64(Y[j * r + t]);
#pragma unroll
        for (int q = 0; q < RB_ROWS; ++q) {
          const double df = fs[q * r + t] - fv;
          e[q] = fma(df, df, e[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < RB_ROWS; ++q) {
        if (ri[q] < 0 || j <= ri[q] || o[q] == 0.0) continue;  // zero pair: not evaluated
        const double v = fabs(sqrt(e[q]) / sqrt(o[q]) - 1.0);
        if (v > best[q]) {  // j increases per lane: ties keep the lowest j
          best[q] = v;
          barg[q] = j;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < RB_ROWS; ++q) {
    for (int s = 16; s; s >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best[q], s);
      const int64_t oa = __shfl_xor_sync(0xffffffffu, barg[q], s);
      if (ov > best[q] || (ov == best[q] && oa < barg[q])) {
        best[q] = ov;
        barg[q] = oa;
      }
    }
    if (lane == 0) {
      w_max[warp][q] = best[q];
      w_arg[warp][q] = barg[q];
    }
  }
  __syncthreads();
  if (threadIdx.x < RB_ROWS) {
    const int q = threadIdx.x;
    double m = -1.0;
    int64_t a = INT64_MAX;
    for (int w = 0; w < RR_THREADS / 32; ++w)
      if (w_max[w][q] > m || (w_max[w][q] == m && w_arg[w][q] < a)) {
        m = w_max[w][q];
        a = w_arg[w][q];
      }
    const int64_t slot = batch * RB_ROWS + q;
    if (slot < nrows)
      out[slot * chunks + chunk] = m >= 0.0 ? RowBest{m, ri[q], a} : RowBest{-1.0, -1, -1};
  }
}

void run_row_refine(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d, const void* Y,
                    adg_dtype yd, int64_t r, const int64_t* rows_dev, int64_t nrows,
                    RowBest* out_dev, int64_t* chunks_per_row_out) {
  const size_t shb = sizeof(double) * (size_t)(RB_ROWS * (d + r));
  if (nrows >= 2 && shb <= 200 * 1024) {
    const int64_t chunks = (n + RB_CHUNK - 1) / RB_CHUNK;
    *chunks_per_row_out = chunks;
    const int64_t batches = (nrows + RB_ROWS - 1) / RB_ROWS;
    ADG_DISPATCH_DTYPE(xd, TO, {
      ADG_DISPATCH_DTYPE(yd, TE, {
        const bool vec = d % 4 == 0 && (reinterpret_cast<uintptr_t>(X) % (4 * sizeof(TO))) == 0;
        auto kern = vec ? row_refine_batch_kernel<TO, TE, true> : row_refine_batch_kernel<TO, TE, false>;
        ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shb));
        kern<<<(unsigned)(batches * chunks), RR_THREADS, shb, ctx->stream>>>(
            (const TO*)X, n, d, (const TE*)Y, r, rows_dev, nrows, out_dev, chunks);
      });
    });
    after_launch(ctx);
    return;
  }
  const int64_t cpr = row_refine_chunks(n);
  *chunks_per_row_out = cpr;
  if (nrows == 0) return;
  const size_t sh = sizeof(double) * (size_t)(d + r);
  ADG_DISPATCH_DTYPE(xd, TO, {
    ADG_DISPATCH_DTYPE(yd, TE, {
      const bool vec = std::is_same<TO, float>::value && d % 4 == 0 &&
                       (reinterpret_cast<uintptr_t>(X) % 16) == 0;
      auto kern = vec ? row_refine_kernel<TO, TE, true> : row_refine_kernel<TO, TE, false>;
      if (sh > 48 * 1024) ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
      kern<<<(unsigned)(nrows * cpr), RR_THREADS, sh, ctx->stream>>>(
          (const TO*)X, n, d, (const TE*)Y, r, rows_dev, out_dev, cpr, 0, rr_chunk(n));
    });
  });
  after_launch(ctx);
}

void run_row_refine_chunks(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t n, int64_t d,
                           const void* Y, adg_dtype yd, int64_t r, const int64_t* row_dev,
                           int64_t chunk0, int64_t chunk1, RowBest* out_dev) {
  if (chunk1 <= chunk0) return;
  const size_t sh = sizeof(double) * (size_t)(d + r);
  ADG_DISPATCH_DTYPE(xd, TO, {
    ADG_DISPATCH_DTYPE(yd, TE, {
      const bool vec = std::is_same<TO, float>::value && d % 4 == 0 &&
                       (reinterpret_cast<uintptr_t>(X) % 16) == 0;
      auto kern = vec ? row_refine_kernel<TO, TE, true> : row_refine_kernel<TO, TE, false>;
      if (sh > 48 * 1024) ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
      kern<<<(unsigned)(chunk1 - chunk0), RR_THREADS, sh, ctx->stream>>>(
          (const TO*)X, n, d, (const TE*)Y, r, row_dev, out_dev, chunk1 - chunk0, chunk0, rr_chunk(n));
    });
  });
  after_launch(ctx);
}

// ------------------------------------------------------ listed pairs
// Exact value of each listed (i, j) pair; -1 marks a zero pair.  One warp per pair.
template <typename TO, typename TE>
__global__ void pair_list_kernel(const TO* __restrict__ X, int64_t d, const TE* __restrict__ Y,
                                 int64_t r, const uint32_t* __restrict__ pairs, int64_t count,
                                 double* __restrict__ values) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= count) return;
  const int64_t i = pairs[2 * w], j = pairs[2 * w + 1];
  ADG_DCHECK(i < j);
  double o = 0.0, e = 0.0;
  for (int64_t t = lane; t < d; t += 32) {
    const double df = to_f64(X[i * d + t]) - to_f64(X[j * d + t]);
    o = fma(df, df, o);
  }
  for (int64_t t = lane; t < r; t += 32) {
    const double df = to_f64(Y[i * r + t]) - to_f64(Y[j * r + t]);
    e = fma(df, df, e);
  }
  for (int s = 16; s; s >>= 1) {
    o += __shfl_xor_sync(0xffffffffu, o, s);
    e += __shfl_xor_sync(0xffffffffu, e, s);
  }
  if (lane == 0) values[w] = (o == 0.0) ? -1.0 : fabs(sqrt(e) / sqrt(o) - 1.0);
}

void run_pair_list(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t d, const void* Y,
                   adg_dtype yd, int64_t r, const uint32_t* pairs_dev, int64_t count,
                   double* values_dev) {
  if (count == 0) return;
  ADG_DISPATCH_DTYPE(xd, TO, {
    ADG_DISPATCH_DTYPE(yd, TE, {
      pair_list_kernel<TO, TE><<<blocks_for(count * 32, 256), 256, 0, ctx->stream>>>(
          (const TO*)X, d, (const TE*)Y, r, pairs_dev, count, values_dev);
    });
  });
  after_launch(ctx);
}

// ------------------------------------------------------- edge list
// Exact binning of the pairs the SCREEN left out of its histogram because
// their screened interval touched a bin edge: entries [0, min(*count, cap))
// (slots holding the 0xFFFFFFFF sentinel are skipped), each pair's value by
// the reference's direct fp64 differences (distortion.cpp:59-75), binned by
// distortion.cpp:81-87 into per-CTA counters flushed to hist (integer adds:
// the result does not depend on the list order).  One warp per pair, 16-byte
// loads of fp32 rows when they are 16-byte aligned.
constexpr int EB_THREADS = 256;

template <typename TO, typename TE, bool VEC>
__global__ void __launch_bounds__(EB_THREADS)
edge_bin_kernel(const TO* __restrict__ X, int64_t d, const TE* __restrict__ Y, int64_t r,
                const uint2* __restrict__ pairs, const unsigned long long* __restrict__ count,
                int64_t cap, int bins, double hist_max, unsigned long long* __restrict__ hist,
                bool global_hist, unsigned long long* __restrict__ binned,
                unsigned long long* __restrict__ near_count, int64_t near_cap) {
  extern __shared__ unsigned int eb_hist[];
  __shared__ unsigned int eb_count;
  if (threadIdx.x == 0) eb_count = 0;
  if (!global_hist)
    for (int b = threadIdx.x; b <= bins; b += EB_THREADS) eb_hist[b] = 0;
  __syncthreads();
  const unsigned long long c = *count;
  const int64_t total = (int64_t)(c < (unsigned long long)cap ? c : (unsigned long long)cap);
  const int lane = threadIdx.x & 31;
  if (c > (unsigned long long)cap && blockIdx.x == 0 && threadIdx.x == 0 && near_count)
    atomicMax(near_count, (unsigned long long)(near_cap + 1));  // -> chunked redo in the finalize
  const int64_t nw = (int64_t)gridDim.x * (EB_THREADS / 32);
  for (int64_t w = ((int64_t)blockIdx.x * EB_THREADS + threadIdx.x) >> 5; w < total; w += nw) {
    const uint2 pr = pairs[w];
    if (pr.x == 0xFFFFFFFFu) continue;  // unused slot of a reserved chunk (warp-uniform)
    const int64_t i = pr.x, j = pr.y;
    ADG_DCHECK(i < j);
    double o = 0.0, e = 0.0;
    if constexpr (VEC) {
      const float4* xi = reinterpret_cast<const float4*>(X + i * d);
      const float4* xj = reinterpret_cast<const float4*>(X + j * d);
      for (int64_t t = lane; t < d / 4; t += 32) {
        const float4 a = __ldg(xi + t), b = __ldg(xj + t);
        double df = (double)a.x - (double)b.x;
        o = fma(df, df, o);
        df = (double)a.y - (double)b.y;
        o = fma(df, df, o);
        df = (double)a.z - (double)b.z;
        o = fma(df, df, o);
        df = (double)a.w - (double)b.w;
        o = fma(df, df, o);
      }
    } else {
      for (int64_t t = lane; t < d; t += 32) {
        const double df = to_f64(X[i * d + t]) - to_f64(X[j * d + t]);
        o = fma(df, df, o);
      }
    }
    for (int64_t t = lane; t < r; t += 32) {
      const double df = to_f64(Y[i * r + t]) - to_f64(Y[j * r + t]);
      e = fma(df, df, e);
    }
    for (int s = 16; s; s >>= 1) {
      o += __shfl_xor_sync(0xffffffffu, o, s);
      e += __shfl_xor_sync(0xffffffffu, e, s);
    }
    // o == 0 cannot reach this list (such pairs screen as near-coincident)
    if (lane == 0 && o != 0.0) {
      const int b = bin_of(fabs(sqrt(e) / sqrt(o) - 1.0), bins, hist_max);
      if (global_hist)
        atomicAdd(&hist[b], 1ull);
      else
        atomicAdd(&eb_hist[b], 1u);
      atomicAdd(&eb_count, 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && eb_count) atomicAdd(binned, (unsigned long long)eb_count);
  if (!global_hist)
    for (int b = threadIdx.x; b <= bins; b += EB_THREADS)
      if (eb_hist[b]) atomicAdd(&hist[b], (unsigned long long)eb_hist[b]);
}

void run_edge_bin(adg_ctx* ctx, const void* X, adg_dtype xd, int64_t d, const void* Y,
                  adg_dtype yd, int64_t r, const uint2* pairs_dev,
                  const unsigned long long* count_dev, int64_t cap, int bins, double hist_max,
                  unsigned long long* hist_dev, unsigned long long* binned_dev,
                  unsigned long long* near_count_dev, int64_t near_cap) {
  if (cap <= 0) return;
  const size_t sh = (size_t)(bins + 1) * sizeof(unsigned);
  const bool global_hist = sh > 160 * 1024;
  const unsigned grid = (unsigned)(4 * ctx->num_sms);  // grid-stride over the device-side count
  ADG_DISPATCH_DTYPE(xd, TO, {
    ADG_DISPATCH_DTYPE(yd, TE, {
      const bool vec = std::is_same<TO, float>::value && d % 4 == 0 &&
                       (reinterpret_cast<uintptr_t>(X) & 15) == 0;
      auto kern = vec ? edge_bin_kernel<TO, TE, true> : edge_bin_kernel<TO, TE, false>;
      if (!global_hist && sh > 48 * 1024)
        ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
      kern<<<grid, EB_THREADS, global_hist ? 0 : sh, ctx->stream>>>(
          (const TO*)X, d, (const TE*)Y, r, pairs_dev, count_dev, cap, bins, hist_max, hist_dev,
          global_hist, binned_dev, near_count_dev, near_cap);
    });
  });
  after_launch(ctx);
}

}  // namespace adg
