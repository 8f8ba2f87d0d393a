// adg_spectral.cu -- the data-aware step on the GPU (sm_100a, fp64).
//
// Reference: proj/src/spectral.cpp:21-101 (exact_top_svd = Eigen BDCSVD of the
// centred n x d cloud; randomized_top_svd = Halko range finder with
// HouseholderQR).  Here both go through the d x d Gram C = Xc^T Xc built with
// fp64 accumulation (the cut gaps of the BASELINE configs need it, SURVEY.md
// 7.3), then:
//   exact:      blocked subspace iteration on C with block b = 2s + 32,
//               CholeskyQR2 re-orthonormalisation and a Rayleigh-Ritz step
//               (one-CTA parallel cyclic Jacobi on the b x b projection) every
//               iteration, stopped on the Ritz residuals; small d goes straight
//               to a full Jacobi of C.  Singular values are ||Xc v|| (one-sided,
//               so tiny ones keep their relative accuracy).
//   randomized: only span(Q) of the reference's range finder matters, so
//               B^T B = C Z (Z^T C Z)^+ Z^T C with Z = orth(C^q Omega), Omega the
//               reference's SeededRng normals (adg_embed.cu), solved by two small
//               Jacobi eigenproblems.
// Rows are sign-normalised exactly like normalize_row_signs
// (spectral.cpp:21-27): the first max-|.| entry is made positive.
#include "adg_spectral.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace adg {

// ----------------------------------------------------------- fp64 GEMM
constexpr int DG_T = 64, DG_K = 16, DG_THREADS = 256;

// grid.z > 1: split-K -- slice z covers K rows [z kslice, (z+1) kslice) and
// writes its raw product to part[z] (M x N); dgemm_splitk_reduce sums the
// slices in z order (deterministic) and applies alpha / beta.
// The product runs on the fp64 tensor cores (DMMA m8n8k4): 8 warps as 4 x 2
// over the 64 x 64 tile (16 x 32 per warp = 2 x 4 fragments); a 16-deep K
// chunk is staged in shared memory (rows padded to 68 doubles: conflict-free
// fragment loads) and the next chunk is loaded into registers under the
// current chunk's MMAs (these products are latency-bound).
constexpr int DG_STR = DG_T + 4, DG_LD = DG_T * DG_K / DG_THREADS;

__device__ __forceinline__ void dg_dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(DG_THREADS)
dgemm_kernel(int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A, int64_t lda,
             const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C,
             int64_t ldc, int64_t kslice, double* __restrict__ part) {
  __shared__ double As[DG_K][DG_STR];
  __shared__ double Bs[DG_K][DG_STR];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int64_t m0 = (int64_t)blockIdx.y * DG_T, n0 = (int64_t)blockIdx.x * DG_T;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int64_t kbeg = part ? (int64_t)blockIdx.z * kslice : 0;
  const int64_t kend = part ? (kbeg + kslice < K ? kbeg + kslice : K) : K;
  double ra[DG_LD], rb[DG_LD];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int t = 0; t < DG_LD; ++t) {
      const int e = tid + t * DG_THREADS;
      int mm, kk;
      if (TA) { mm = e % DG_T; kk = e / DG_T; } else { kk = e % DG_K; mm = e / DG_K; }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      ra[t] = (gm < M && gk < kend) ? (TA ? A[gk * lda + gm] : A[gm * lda + gk]) : 0.0;
      int nn, kb;
      if (TB) { kb = e % DG_K; nn = e / DG_K; } else { nn = e % DG_T; kb = e / DG_T; }
      const int64_t gn = n0 + nn, gkb = k0 + kb;
      rb[t] = (gn < N && gkb < kend) ? (TB ? B[gn * ldb + gkb] : B[gkb * ldb + gn]) : 0.0;
    }
  };
  if (kbeg < kend) fetch(kbeg);
  for (int64_t k0 = kbeg; k0 < kend; k0 += DG_K) {
#pragma unroll
    for (int t = 0; t < DG_LD; ++t) {
      const int e = tid + t * DG_THREADS;
      if (TA) As[e / DG_T][e % DG_T] = ra[t]; else As[e % DG_K][e / DG_K] = ra[t];
      if (TB) Bs[e % DG_K][e / DG_K] = rb[t]; else Bs[e / DG_T][e % DG_T] = rb[t];
    }
    __syncthreads();
    if (k0 + DG_K < kend) fetch(k0 + DG_K);
#pragma unroll
    for (int ks = 0; ks < DG_K / 4; ++ks) {
      const int kr = ks * 4 + (lane & 3);
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = As[kr][wm * 16 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[kr][wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dg_dmma(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t gm = m0 + wm * 16 + i * 8 + (lane >> 2);
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gn = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
        if (gn >= N) continue;
        if (part) {
          part[((int64_t)blockIdx.z * M + gm) * N + gn] = acc[i][j][h];
          continue;
        }
        const double prev = beta == 0.0 ? 0.0 : beta * C[gm * ldc + gn];
        C[gm * ldc + gn] = alpha * acc[i][j][h] + prev;
      }
  }
}

__global__ void dgemm_splitk_reduce(const double* __restrict__ part, int splits, int64_t M, int64_t N,
                                    double alpha, double beta, double* __restrict__ C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int z = 0; z < splits; ++z) acc += part[z * total + t];
    const int64_t gm = t / N, gn = t % N;
    const double prev = beta == 0.0 ? 0.0 : beta * C[gm * ldc + gn];
    C[gm * ldc + gn] = alpha * acc + prev;
  }
}

void dgemm(adg_ctx* ctx, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
           const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
           int64_t ldc) {
  if (M <= 0 || N <= 0) return;
  const int64_t tiles = ((N + DG_T - 1) / DG_T) * ((M + DG_T - 1) / DG_T);
  // small output grids (tall-skinny products of the subspace iteration) split
  // K over enough CTAs to fill the SMs: these launches are latency-bound
  int64_t splits = 1, kslice = K;
  if (tiles < ctx->num_sms / 2 && K >= 8 * DG_K) {
    splits = std::min<int64_t>((ctx->num_sms + tiles - 1) / tiles, K / (4 * DG_K));
    kslice = (K + splits - 1) / splits;
    kslice = (kslice + DG_K - 1) / DG_K * DG_K;
    splits = (K + kslice - 1) / kslice;
  }
  DevBuf<double> part(splits > 1 ? (size_t)(splits * M * N) : 0, ctx->stream);
  double* pp = splits > 1 ? part.ptr : nullptr;
  dim3 grid((unsigned)((N + DG_T - 1) / DG_T), (unsigned)((M + DG_T - 1) / DG_T), (unsigned)splits);
  if (!ta && !tb)
    dgemm_kernel<false, false><<<grid, DG_THREADS, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kslice, pp);
  else if (ta && !tb)
    dgemm_kernel<true, false><<<grid, DG_THREADS, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kslice, pp);
  else if (!ta && tb)
    dgemm_kernel<false, true><<<grid, DG_THREADS, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kslice, pp);
  else
    dgemm_kernel<true, true><<<grid, DG_THREADS, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, kslice, pp);
  after_launch(ctx);
  if (splits > 1) {
    dgemm_splitk_reduce<<<blocks_for(M * N, 256, 4 * ctx->num_sms), 256, 0, ctx->stream>>>(
        pp, (int)splits, M, N, alpha, beta, C, ldc);
    after_launch(ctx);
  }
}

// --------------------------------------------------------------- Gram
// Centred fp64 Gram C = Xc^T Xc on the fp64 tensor cores (DMMA m8n8k4,
// IEEE fp64 products and sums).  A CTA owns one 128 x 128 tile of the upper
// block triangle and one slice of rows (split K, summed afterwards in a fixed
// order, so the result does not depend on scheduling): each 32-row chunk of X
// is widened to fp64 and centred while it is staged in shared memory (rows
// padded to 132 doubles: the 4 k-rows x 8 columns of a fragment load hit 16
// distinct bank pairs per half-warp), and the next chunk's loads are issued
// before the current chunk's MMAs.  8 warps as 2 x 4, a 64 x 32 warp tile =
// 8 x 4 fragments, 12 shared loads per 32 DMMAs.
constexpr int GM_T = 128, GM_K = 32, GM_STR = GM_T + 4, GM_THREADS = 256;
constexpr int GM_LD = GM_K * GM_T / GM_THREADS;  // elements a thread stages per operand

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename T>
__global__ void __launch_bounds__(GM_THREADS, 1)
gram_partial_kernel(const T* __restrict__ X, int64_t n, int64_t d, const double* __restrict__ mean,
                    int64_t rows_per_split, double* __restrict__ part) {
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  if (bi > bj) return;
  extern __shared__ double gsm[];
  double* As = gsm;                     // GM_K x GM_STR
  double* Bs = gsm + GM_K * GM_STR;     // GM_K x GM_STR
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int64_t m0 = bi * GM_T, n0 = bj * GM_T;
  const int64_t r0 = (int64_t)blockIdx.z * rows_per_split;
  const int64_t r1 = r0 + rows_per_split < n ? r0 + rows_per_split : n;
  // staging: column tid % 128 of the tile, rows tid / 128 + 2 t
  const int col = tid & (GM_T - 1), kr0 = tid >> 7;
  const int64_t ga = m0 + col, gb = n0 + col;
  const bool va_ok = ga < d, vb_ok = gb < d;
  const double mua = (mean && va_ok) ? mean[ga] : 0.0, mub = (mean && vb_ok) ? mean[gb] : 0.0;
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // the next chunk is held raw (input type) and widened at the shared store,
  // so nothing consumes the loads before the MMAs that hide them
  T xa[GM_LD], xb[GM_LD];
  unsigned live = 0;  // bit t: row kr0 + 2 t of the chunk exists
  auto fetch = [&](int64_t k0) {
    live = 0;
#pragma unroll
    for (int t = 0; t < GM_LD; ++t) {
      const int64_t gk = k0 + kr0 + 2 * t;
      const bool rk = gk < r1;
      live |= rk ? (1u << t) : 0u;
      const int64_t row = rk ? gk : r0;  // an in-range row; masked at the store
      xa[t] = X[row * d + (va_ok ? ga : 0)];
      xb[t] = X[row * d + (vb_ok ? gb : 0)];
    }
  };
  if (r0 < r1) fetch(r0);
  for (int64_t k0 = r0; k0 < r1; k0 += GM_K) {
#pragma unroll
    for (int t = 0; t < GM_LD; ++t) {
      const bool rk = (live >> t) & 1u;
      As[(kr0 + 2 * t) * GM_STR + col] = (rk && va_ok) ? to_f64(xa[t]) - mua : 0.0;
      Bs[(kr0 + 2 * t) * GM_STR + col] = (rk && vb_ok) ? to_f64(xb[t]) - mub : 0.0;
    }
    __syncthreads();
    if (k0 + GM_K < r1) fetch(k0 + GM_K);  // in flight under the MMAs below
#pragma unroll
    for (int ks = 0; ks < GM_K / 4; ++ks) {
      const int kr = ks * 4 + (lane & 3);
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = As[kr * GM_STR + wm * 64 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[kr * GM_STR + wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
  double* P = part + (int64_t)blockIdx.z * d * d;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gm = m0 + wm * 64 + i * 8 + (lane >> 2);
    if (gm >= d) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gn = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
        if (gn < d) P[gm * d + gn] = acc[i][j][h];
      }
  }
}

__global__ void gram_reduce_kernel(const double* __restrict__ part, int64_t splits, int64_t d,
                                   double* __restrict__ G) {
  const int64_t total = d * d;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / d, j = t % d;
    const int64_t bi = i / GM_T, bj = j / GM_T;
    // the tile holding (i, j) was computed in the upper block triangle
    const int64_t src = (bi <= bj) ? (i * d + j) : (j * d + i);
    double acc = 0.0;
    for (int64_t s = 0; s < splits; ++s) acc += part[s * total + src];
    G[t] = acc;
  }
}

void gram_f64(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d,
              const double* mean, double* G) {
  const int64_t tb = (d + GM_T - 1) / GM_T;
  const int64_t tiles = tb * (tb + 1) / 2;
  // one CTA per SM (acc = 64 doubles per lane): ~4 waves of upper tiles
  int64_t splits = std::max<int64_t>(1, (4 * ctx->num_sms + tiles / 2) / tiles);
  // bound the partial workspace to ~1 GiB
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, (int64_t)(1ll << 27) / (d * d)));
  int64_t rows = (n + splits - 1) / splits;
  rows = (rows + GM_K - 1) / GM_K * GM_K;
  splits = std::max<int64_t>(1, (n + rows - 1) / rows);
  DevBuf<double> part((size_t)(splits * d * d), ctx->stream);
  dim3 grid((unsigned)tb, (unsigned)tb, (unsigned)splits);
  const size_t smem = sizeof(double) * 2 * GM_K * GM_STR;
  ADG_DISPATCH_DTYPE(dt, T, {
    ADG_CUDA(cudaFuncSetAttribute(gram_partial_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    gram_partial_kernel<T><<<grid, GM_THREADS, smem, ctx->stream>>>((const T*)X, n, d, mean, rows,
                                                                    part.ptr);
  });
  after_launch(ctx);
  gram_reduce_kernel<<<blocks_for(d * d, 256, 8 * ctx->num_sms), 256, 0, ctx->stream>>>(
      part.ptr, splits, d, G);
  after_launch(ctx);
}

// ------------------------------------------------------ Jacobi (1 CTA)
// Parallel cyclic two-sided Jacobi on a symmetric m x m matrix (round-robin
// ordering: m/2 disjoint rotations per round, m-1 rounds per sweep).
// Rotation per Golub & Van Loan 8.4 (symmetric Schur); a pair is skipped when
// |a_pq| <= 1e-17 sqrt(|a_pp a_qq|) (high relative accuracy).  A is kept in
// shared memory when it fits, V in global.  Output: eigenvalues diag(A).
constexpr int JAC_THREADS = 1024;

// SMEM: 0 A and V in global, 1 A in shared, 2 A and V in shared
template <int SMEM>
__global__ void __launch_bounds__(JAC_THREADS)
jacobi_kernel(double* __restrict__ Ag, double* __restrict__ Vg, int m, int max_sweeps,
              bool init_identity, double* __restrict__ evals, int* __restrict__ info) {
  extern __shared__ double sh[];
  constexpr bool use_smem = SMEM >= 1;
  const int mm = m + (m & 1);  // players incl. a bye for odd m
  const int npairs = mm / 2;
  double* cs = sh;                   // [npairs] c
  double* sn = sh + npairs;          // [npairs] s
  int* pp = reinterpret_cast<int*>(sh + 2 * npairs);  // [npairs]
  int* qq = pp + npairs;                              // [npairs]
  __shared__ int rotated;
  double* A = use_smem ? reinterpret_cast<double*>(reinterpret_cast<char*>(sh) +
                                                    ((size_t)npairs * 24 + 15) / 16 * 16)
                       : Ag;
  double* V = SMEM == 2 ? A + (size_t)m * m : Vg;
  const int tid = threadIdx.x;
  if (use_smem)
    for (int e = tid; e < m * m; e += JAC_THREADS) A[e] = Ag[e];
  if (init_identity)
    for (int e = tid; e < m * m; e += JAC_THREADS) V[e] = (e / m == e % m) ? 1.0 : 0.0;
  else if (SMEM == 2)
    for (int e = tid; e < m * m; e += JAC_THREADS) V[e] = Vg[e];
  __syncthreads();
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < mm - 1; ++round) {
      for (int k = tid; k < npairs; k += JAC_THREADS) {
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + ((pos - 1 + round) % (mm - 1)); };
        int p = player(k), q = player(mm - 1 - k);
        if (p > q) { const int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0;
        if (q < m) {
          const double apq = A[p * m + q];
          const double app = A[p * m + p], aqq = A[q * m + q];
          if (apq != 0.0 && fabs(apq) > 1e-17 * sqrt(fabs(app * aqq))) {
            const double theta = (aqq - app) / (2.0 * apq);
            double t;
            if (fabs(theta) > 1e150)
              t = 0.5 / theta;
            else
              t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
            rotated = 1;
          }
        }
        cs[k] = c;
        sn[k] = s;
        pp[k] = p;
        qq[k] = q < m ? q : -1;
      }
      __syncthreads();
      // A <- A J (columns p, q of every row);  V <- V J
      for (int e = tid; e < m * npairs; e += JAC_THREADS) {
        const int k = e % npairs, r = e / npairs;
        const int q = qq[k];
        if (q < 0 || sn[k] == 0.0) continue;
        const int p = pp[k];
        const double c = cs[k], s = sn[k];
        const double ap = A[r * m + p], aq = A[r * m + q];
        A[r * m + p] = c * ap - s * aq;
        A[r * m + q] = s * ap + c * aq;
        const double vp = V[r * m + p], vq = V[r * m + q];
        V[r * m + p] = c * vp - s * vq;
        V[r * m + q] = s * vp + c * vq;
      }
      __syncthreads();
      // A <- J^T A (rows p, q of every column)
      for (int e = tid; e < m * npairs; e += JAC_THREADS) {
        const int k = e % npairs, col = e / npairs;
        const int q = qq[k];
        if (q < 0 || sn[k] == 0.0) continue;
        const int p = pp[k];
        const double c = cs[k], s = sn[k];
        const double ap = A[p * m + col], aq = A[q * m + col];
        A[p * m + col] = c * ap - s * aq;
        A[q * m + col] = s * ap + c * aq;
      }
      __syncthreads();
      for (int k = tid; k < npairs; k += JAC_THREADS) {
        const int q = qq[k];
        if (q < 0 || sn[k] == 0.0) continue;
        const int p = pp[k];
        A[p * m + q] = 0.0;
        A[q * m + p] = 0.0;
      }
      __syncthreads();
    }
    if (!rotated) break;
  }
  for (int e = tid; e < m; e += JAC_THREADS) evals[e] = A[e * m + e];
  if (use_smem)
    for (int e = tid; e < m * m; e += JAC_THREADS) Ag[e] = A[e];
  if (SMEM == 2)
    for (int e = tid; e < m * m; e += JAC_THREADS) Vg[e] = V[e];
  if (tid == 0 && info) *info = sweep;
}

// The same sweeps with A ping-ponged in shared memory (m <= JPP_MAXM): every
// 2x2 block (row pair, column pair) of a round goes B' = J1^T (B J2) from the
// round's input copy into the other, the exact operation sequence of the
// column-then-row passes above (bit-identical results), with two barriers
// per round instead of four and one read + write of A per round instead of
// two.  V (shared) is updated in the same pass.
constexpr int JPP_MAXM = 92;

__global__ void __launch_bounds__(JAC_THREADS)
jacobi_pp_kernel(double* __restrict__ Ag, double* __restrict__ Vg, int m, int max_sweeps,
                 double* __restrict__ evals, int* __restrict__ info) {
  extern __shared__ double sh[];
  const int mm = m + (m & 1);
  const int npairs = mm / 2;
  double* cs = sh;
  double* sn = sh + npairs;
  int* pp = reinterpret_cast<int*>(sh + 2 * npairs);
  int* qq = pp + npairs;
  __shared__ int rotated;
  // per-index column rotation: new a_j = jc[j] a_j + js[j] a_{jpart[j]}
  double* jc = reinterpret_cast<double*>(reinterpret_cast<char*>(sh) + ((size_t)npairs * 24 + 15) / 16 * 16);
  double* js = jc + m;
  int* jpart = reinterpret_cast<int*>(js + m);
  double* cur = reinterpret_cast<double*>(reinterpret_cast<char*>(jpart) + ((size_t)m * 4 + 15) / 16 * 16);
  double* nxt = cur + (size_t)m * m;
  double* Vt = nxt + (size_t)m * m;  // V transposed: column c of V = row c of Vt
  const int tid = threadIdx.x, lx = tid & 31, wy = tid >> 5;
  constexpr int NW = JAC_THREADS / 32;
  for (int e = tid; e < m * m; e += JAC_THREADS) {
    cur[e] = Ag[e];
    Vt[e] = (e / m == e % m) ? 1.0 : 0.0;
  }
  __syncthreads();
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < mm - 1; ++round) {
      for (int k = tid; k < npairs; k += JAC_THREADS) {
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + ((pos - 1 + round) % (mm - 1)); };
        int p = player(k), q = player(mm - 1 - k);
        if (p > q) { const int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0;
        if (q < m) {
          const double apq = cur[p * m + q];
          const double app = cur[p * m + p], aqq = cur[q * m + q];
          // the round's critical path: one sqrt, one division and one rsqrt
          // (t = tan of the Schur angle from a_pq and a_qq - a_pp directly,
          // skip test squared)
          if (apq != 0.0 && apq * apq > 1e-34 * fabs(app * aqq)) {
            const double dd = aqq - app;
            const double t = (dd >= 0.0 ? 2.0 * apq : -2.0 * apq) /
                             (fabs(dd) + sqrt(fma(dd, dd, 4.0 * apq * apq)));
            c = rsqrt(fma(t, t, 1.0));
            s = t * c;
            rotated = 1;
          }
        }
        cs[k] = c;
        sn[k] = s;
        pp[k] = p;
        qq[k] = q < m ? q : -1;
        jc[p] = c;
        js[p] = -s;
        jpart[p] = q < m ? q : p;
        if (q < m) {
          jc[q] = c;
          js[q] = s;
          jpart[q] = p;
        }
      }
      __syncthreads();
      // A <- J^T A J: a warp per row pair (p1, q1), lanes over contiguous
      // columns j (the column partner is the only scattered read)
      for (int k1 = wy; k1 < npairs; k1 += NW) {
        const int p1 = pp[k1], q1 = qq[k1];
        const double c1 = cs[k1], s1 = sn[k1];
        const bool rot1 = q1 >= 0 && s1 != 0.0;
        const double* rp = cur + p1 * m;
        const double* rq = cur + (q1 >= 0 ? q1 : p1) * m;
        for (int j = lx; j < m; j += 32) {
          const int pj = jpart[j];
          const double cj = jc[j], sj = js[j];
          double bp = rp[j], bq = rq[j];
          if (sj != 0.0) {
            bp = cj * bp + sj * rp[pj];
            bq = cj * bq + sj * rq[pj];
          }
          double np = bp, nq = bq;
          if (rot1) {
            np = c1 * bp - s1 * bq;
            nq = s1 * bp + c1 * bq;
            if (j == q1) np = 0.0;  // the annihilated pair
            if (j == p1) nq = 0.0;
          }
          nxt[p1 * m + j] = np;
          if (q1 >= 0) nxt[q1 * m + j] = nq;
        }
      }
      // V <- V J: rows p, q of V^T, lanes over contiguous entries
      for (int k = wy; k < npairs; k += NW) {
        const int q = qq[k];
        const double sk = sn[k];
        if (q < 0 || sk == 0.0) continue;
        const int p = pp[k];
        const double ck = cs[k];
        double* vp = Vt + p * m;
        double* vq = Vt + q * m;
        for (int r = lx; r < m; r += 32) {
          const double a0 = vp[r], a1 = vq[r];
          vp[r] = ck * a0 - sk * a1;
          vq[r] = sk * a0 + ck * a1;
        }
      }
      __syncthreads();
      double* t = cur;
      cur = nxt;
      nxt = t;
    }
    if (!rotated) break;
  }
  for (int e = tid; e < m; e += JAC_THREADS) evals[e] = cur[e * m + e];
  for (int e = tid; e < m * m; e += JAC_THREADS) {
    Ag[e] = cur[e];
    Vg[e] = Vt[(e % m) * m + e / m];
  }
  if (tid == 0 && info) *info = sweep;
}

// ------------------------------------------------ Jacobi (whole grid)
// The same parallel cyclic Jacobi (round-robin pairs, Golub & Van Loan 8.4
// rotations, the same skip rule and sweep test) for large m, over every SM:
// in one round the m/2 pairs are disjoint, so each 2x2 block of A (row pair,
// column pair) is transformed independently, B' = J1^T (B J2), from the
// round's input buffer into the other (ping-pong), and V's column pairs in
// place.  Every CTA derives all the round's rotations itself (shared
// memory), so a round costs one grid barrier; every CTA sees the same
// rotations, so all leave the sweep loop together.
constexpr int JG_THREADS = 512;

struct GridBarrier {
  unsigned count, gen;
};

__device__ __forceinline__ void grid_barrier(GridBarrier* gb, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = &gb->gen;
    const unsigned g = *vgen;
    __threadfence();
    if (atomicAdd(&gb->count, 1u) == nblocks - 1) {
      atomicExch(&gb->count, 0u);
      __threadfence();
      atomicAdd(&gb->gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(JG_THREADS)
jacobi_grid_kernel(double* __restrict__ A0, double* __restrict__ A1, double* __restrict__ V, int m,
                   int max_sweeps, double* __restrict__ evals, GridBarrier* gb,
                   int* __restrict__ result_buf) {
  extern __shared__ double jsm[];
  const int mm = m + (m & 1), npairs = mm / 2;
  double* cs = jsm;               // [npairs]
  double* sn = cs + npairs;       // [npairs]
  int* pp = reinterpret_cast<int*>(sn + npairs);  // [npairs]
  int* qq = pp + npairs;                          // [npairs] (-1: bye)
  __shared__ int any_rot;
  const int tid = threadIdx.x;
  const int64_t gtid = (int64_t)blockIdx.x * JG_THREADS + tid;
  const int64_t gstride = (int64_t)gridDim.x * JG_THREADS;
  for (int64_t e = gtid; e < (int64_t)m * m; e += gstride) V[e] = (e / m == e % m) ? 1.0 : 0.0;
  grid_barrier(gb, gridDim.x);  // V is updated by other CTAs from round 0 on
  double* cur = A0;
  double* nxt = A1;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) any_rot = 0;
    __syncthreads();
    int sweep_rot = 0;
    for (int round = 0; round < mm - 1; ++round) {
      // the round's rotations, from `cur` (written by the previous round)
      for (int k = tid; k < npairs; k += JG_THREADS) {
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + ((pos - 1 + round) % (mm - 1)); };
        int p = player(k), q = player(mm - 1 - k);
        if (p > q) { const int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0;
        if (q < m) {
          const double apq = __ldcg(&cur[(int64_t)p * m + q]);
          const double app = __ldcg(&cur[(int64_t)p * m + p]), aqq = __ldcg(&cur[(int64_t)q * m + q]);
          if (apq != 0.0 && fabs(apq) > 1e-17 * sqrt(fabs(app * aqq))) {
            const double theta = (aqq - app) / (2.0 * apq);
            double t;
            if (fabs(theta) > 1e150)
              t = 0.5 / theta;
            else
              t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
            any_rot = 1;
          }
        }
        cs[k] = c;
        sn[k] = s;
        pp[k] = p;
        qq[k] = q < m ? q : -1;
      }
      __syncthreads();
      sweep_rot |= any_rot;
      const int64_t nblk = (int64_t)npairs * npairs;
      const int64_t total = nblk + (int64_t)m * npairs;
      for (int64_t w = gtid; w < total; w += gstride) {
        if (w < nblk) {
          const int k1 = (int)(w / npairs), k2 = (int)(w % npairs);
          const int p1 = pp[k1], q1 = qq[k1], p2 = pp[k2], q2 = qq[k2];
          const double c1 = cs[k1], s1 = sn[k1], c2 = cs[k2], s2 = sn[k2];
          // B J2 (columns p2, q2 of rows p1, q1), then J1^T (rows), as A J then J^T A
          double b00 = __ldcg(&cur[(int64_t)p1 * m + p2]), b01 = q2 >= 0 ? __ldcg(&cur[(int64_t)p1 * m + q2]) : 0.0;
          double b10 = q1 >= 0 ? __ldcg(&cur[(int64_t)q1 * m + p2]) : 0.0;
          double b11 = (q1 >= 0 && q2 >= 0) ? __ldcg(&cur[(int64_t)q1 * m + q2]) : 0.0;
          if (q2 >= 0 && s2 != 0.0) {
            const double x0 = c2 * b00 - s2 * b01, y0 = s2 * b00 + c2 * b01;
            const double x1 = c2 * b10 - s2 * b11, y1 = s2 * b10 + c2 * b11;
            b00 = x0; b01 = y0; b10 = x1; b11 = y1;
          }
          if (q1 >= 0 && s1 != 0.0) {
            const double x0 = c1 * b00 - s1 * b10, x1 = c1 * b01 - s1 * b11;
            const double y0 = s1 * b00 + c1 * b10, y1 = s1 * b01 + c1 * b11;
            b00 = x0; b01 = x1; b10 = y0; b11 = y1;
          }
          if (k1 == k2 && q1 >= 0 && s1 != 0.0) b01 = b10 = 0.0;  // the annihilated pair
          nxt[(int64_t)p1 * m + p2] = b00;
          if (q2 >= 0) nxt[(int64_t)p1 * m + q2] = b01;
          if (q1 >= 0) nxt[(int64_t)q1 * m + p2] = b10;
          if (q1 >= 0 && q2 >= 0) nxt[(int64_t)q1 * m + q2] = b11;
        } else {
          const int64_t v = w - nblk;
          const int r = (int)(v / npairs), k = (int)(v % npairs);
          const int p = pp[k], q = qq[k];
          const double s = sn[k];
          if (q < 0 || s == 0.0) continue;
          const double c = cs[k];
          const double vp = __ldcg(&V[(int64_t)r * m + p]), vq = __ldcg(&V[(int64_t)r * m + q]);
          V[(int64_t)r * m + p] = c * vp - s * vq;
          V[(int64_t)r * m + q] = s * vp + c * vq;
        }
      }
      grid_barrier(gb, gridDim.x);
      double* t = cur;
      cur = nxt;
      nxt = t;
    }
    if (!sweep_rot) break;
  }
  for (int64_t e = gtid; e < m; e += gstride) evals[e] = __ldcg(&cur[e * m + e]);
  if (gtid == 0 && result_buf) *result_buf = sweep;
}

// CholeskyQR step for large b over the whole grid (cooperative launch): G +
// shift I = R^T R in global memory (L2-resident), one grid barrier per
// elimination step (Schur updates with the unscaled pivot row), then every
// row of Q solved in place, x R = q, one warp per row.
__global__ void __launch_bounds__(JG_THREADS)
chol_trsm_grid_kernel(double* __restrict__ G, int b, double shift_coef, double* __restrict__ Q,
                      int64_t rows, double* __restrict__ rinv, int* __restrict__ info,
                      GridBarrier* gb) {
  const int tid = threadIdx.x;
  const int64_t gtid = (int64_t)blockIdx.x * JG_THREADS + tid;
  const int64_t gstride = (int64_t)gridDim.x * JG_THREADS;
  __shared__ double shift;
  if (tid == 0) {
    double mx = 0.0;
    for (int e = 0; e < b; ++e) mx = fmax(mx, __ldcg(&G[(int64_t)e * b + e]));
    shift = shift_coef * mx;
  }
  __syncthreads();
  grid_barrier(gb, gridDim.x);  // every CTA has read the diagonal
  for (int64_t e = gtid; e < b; e += gstride) G[e * b + e] = __ldcg(&G[e * b + e]) + shift;
  grid_barrier(gb, gridDim.x);
  for (int k = 0; k < b; ++k) {
    const double piv = __ldcg(&G[(int64_t)k * b + k]);
    const double ipiv = piv > 0.0 ? 1.0 / piv : 1.0;
    const int64_t rem = b - k - 1;
    for (int64_t e = gtid; e < rem * rem; e += gstride) {
      const int i = k + 1 + (int)(e / rem), j = k + 1 + (int)(e % rem);
      if (j >= i)
        G[(int64_t)i * b + j] = fma(-__ldcg(&G[(int64_t)k * b + i]) * ipiv, __ldcg(&G[(int64_t)k * b + j]),
                                    __ldcg(&G[(int64_t)i * b + j]));
    }
    grid_barrier(gb, gridDim.x);
  }
  for (int64_t k = gtid; k < b; k += gstride) {
    const double piv = __ldcg(&G[k * b + k]);
    if (!(piv > 0.0)) atomicExch(info, 1);
    rinv[k] = piv > 0.0 ? 1.0 / sqrt(piv) : 1.0;
  }
  grid_barrier(gb, gridDim.x);
  for (int64_t e = gtid; e < (int64_t)b * b; e += gstride) {
    const int64_t i = e / b, j = e % b;
    if (j > i) G[e] = __ldcg(&G[e]) * __ldcg(&rinv[i]);
  }
  grid_barrier(gb, gridDim.x);
  // rows of Q: a warp per row, lanes over the remaining columns
  const int lane = tid & 31;
  const int64_t warp = gtid >> 5, nwarps = gstride >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    double* q = Q + r * b;
    for (int j = 0; j < b; ++j) {
      const double xj = q[j] * __ldcg(&rinv[j]);
      __syncwarp();
      if (lane == 0) q[j] = xj;
      for (int l = j + 1 + lane; l < b; l += 32) q[l] = fma(-xj, __ldcg(&G[(int64_t)j * b + l]), q[l]);
      __syncwarp();
    }
  }
}

// Sort eigenpairs descending (stable: ties keep the lower index) and emit the
// first `keep` eigenvectors as columns of Vout (m x keep) and values.
__global__ void sort_eig_kernel(const double* __restrict__ evals, const double* __restrict__ V, int m,
                                int keep, double* __restrict__ vals_out, double* __restrict__ Vout) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const double ei = evals[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double ej = evals[j];
      rank += (ej > ei) || (ej == ei && j < i);
    }
    if (rank < keep) {
      vals_out[rank] = ei;
      for (int r = 0; r < m; ++r) Vout[(int64_t)r * keep + rank] = V[(int64_t)r * m + i];
    }
  }
}

struct Eig {
  DevBuf<double> vals, vecs;  // vecs: m x keep (column k = k-th largest)
};

static void sym_eig(adg_ctx* ctx, const double* A_in, int m, int keep, Eig& out) {
  DevBuf<double> A((size_t)m * m, ctx->stream), V((size_t)m * m, ctx->stream),
      ev((size_t)m, ctx->stream);
  ADG_CUDA(cudaMemcpyAsync(A.ptr, A_in, sizeof(double) * m * m, cudaMemcpyDeviceToDevice,
                           ctx->stream));
  const int mm = m + (m & 1);
  const int npairs = mm / 2;
  const size_t head = ((size_t)npairs * 24 + 15) / 16 * 16;  // c, s (double) + p, q (int)
  const size_t mat = sizeof(double) * (size_t)m * m;
  const size_t cap = 220 * 1024;
  auto go = [&](auto kern, size_t sh) {
    ADG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(sh, 48 * 1024)));
    kern<<<1, JAC_THREADS, sh, ctx->stream>>>(A.ptr, V.ptr, m, 60, true, ev.ptr, nullptr);
  };
  const size_t pp_head = head + ((size_t)m * 16 + 15) / 16 * 16 + ((size_t)m * 4 + 15) / 16 * 16;
  if (m <= JPP_MAXM && pp_head + 3 * mat <= cap) {
    ADG_CUDA(cudaFuncSetAttribute(jacobi_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(pp_head + 3 * mat, 48 * 1024)));
    DevBuf<int> sw(1, ctx->stream);
    jacobi_pp_kernel<<<1, JAC_THREADS, pp_head + 3 * mat, ctx->stream>>>(A.ptr, V.ptr, m, 60, ev.ptr, sw.ptr);
    if (std::getenv("ADG_FIT_PROFILE")) {
      int hs = 0;
      ADG_CUDA(cudaMemcpyAsync(&hs, sw.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      ADG_CUDA(cudaStreamSynchronize(ctx->stream));
      std::fprintf(stderr, "[fit] jacobi m=%d sweeps=%d\n", m, hs);
    }
  } else if (head + 2 * mat <= cap) {
    go(jacobi_kernel<2>, head + 2 * mat);
  } else if (m <= 128 && head + mat <= cap) {
    go(jacobi_kernel<1>, head + mat);
  } else {
    // large m: the whole grid, one cooperative launch (co-residency guaranteed)
    DevBuf<double> A1((size_t)m * m, ctx->stream);
    DevBuf<GridBarrier> gb(1, ctx->stream);
    gb.zero();
    const size_t sh = (size_t)npairs * (2 * sizeof(double) + 2 * sizeof(int));
    ADG_CUDA(cudaFuncSetAttribute(jacobi_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(sh, 48 * 1024)));
    int per_sm = 0;
    ADG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_grid_kernel, JG_THREADS, sh));
    ADG_REQUIRE(per_sm >= 1, "sym_eig: grid Jacobi cannot be resident");
    double* a0 = A.ptr;
    double* a1 = A1.ptr;
    double* vp = V.ptr;
    int mm_ = m, sweeps = 60;
    double* evp = ev.ptr;
    GridBarrier* gbp = gb.ptr;
    int* nullp = nullptr;
    void* args[] = {&a0, &a1, &vp, &mm_, &sweeps, &evp, &gbp, &nullp};
    ADG_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_grid_kernel, dim3((unsigned)ctx->num_sms),
                                         dim3(JG_THREADS), args, sh, ctx->stream));
  }
  after_launch(ctx);
  out.vals.alloc((size_t)keep, ctx->stream);
  out.vecs.alloc((size_t)m * keep, ctx->stream);
  sort_eig_kernel<<<blocks_for(m, 128), 128, 0, ctx->stream>>>(ev.ptr, V.ptr, m, keep,
                                                               out.vals.ptr, out.vecs.ptr);
  after_launch(ctx);
}

// -------------------------------------------------- Cholesky QR
// Fused CholeskyQR step for b <= CT_MAXB: every CTA factors G + shift I =
// R^T R in shared memory (redundantly -- b is small) and then solves its own
// 32 rows of Q in place, x R = q by forward substitution, right-looking so
// each row's FMAs are independent across the remaining columns.
constexpr int CT_ROWS = 8, CT_MAXB = 112, CT_THREADS = 256;

__global__ void __launch_bounds__(CT_THREADS)
chol_trsm_kernel(const double* __restrict__ Gg, int b, double shift_coef, double* __restrict__ Q,
                 int64_t rows, int* __restrict__ info) {
  extern __shared__ double sm[];
  double* G = sm;                               // b x b
  double* qs = sm + (size_t)b * b;              // CT_ROWS x (b + 1)
  double* rinv = qs + (size_t)CT_ROWS * (b + 1);  // b
  __shared__ double rowbuf[2 * CT_MAXB];         // pivot rows (double-buffered)
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5, nwy = CT_THREADS / 32;
  __shared__ int bad;
  __shared__ double shift;
  for (int e = tid; e < b * b; e += CT_THREADS) G[e] = Gg[e];
  const int64_t r0 = (int64_t)blockIdx.x * CT_ROWS;
  for (int e = tid; e < CT_ROWS * b; e += CT_THREADS) {
    const int rr = e / b, c = e % b;
    qs[rr * (b + 1) + c] = (r0 + rr < rows) ? Q[(r0 + rr) * b + c] : 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int e = 0; e < b; ++e) mx = fmax(mx, G[e * b + e]);
    shift = shift_coef * mx;
  }
  __syncthreads();
  for (int e = tid; e < b; e += CT_THREADS) G[e * b + e] += shift;
  __syncthreads();
  // Schur complements with the unscaled pivot row, G_ij -= G_ki G_kj / G_kk
  // for k < i <= j (rows scaled by 1/sqrt(G_kk) after).  A thread keeps its
  // elements (rows ty + 16 a, columns tx + 16 c) in registers for the whole
  // factorisation; the owners of row k+1 publish it to a double-buffered
  // shared row as soon as step k has updated it, so a step is one barrier and
  // ~2 NA shared loads per thread (the shared-memory re-read of every element
  // per step was the kernel's bound).  Same FMAs in the same order as a
  // shared-memory right-looking update.
  {
    const int ty = tid >> 4, tx = tid & 15;
    constexpr int NA = (CT_MAXB + 15) / 16;
    static_assert(NA == 7, "publish switch below covers 7 row groups");
    double v[NA][NA];
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int c = 0; c < NA; ++c) {
        const int i = ty + 16 * a, j = tx + 16 * c;
        v[a][c] = (j >= i && j < b) ? G[i * b + j] : 0.0;
      }
    // pivot rows: [b, CT_MAXB) stays zero, so the loads below need no bounds
    // test (branch-free: selects, not predicated loads)
    for (int e = tid; e < 2 * CT_MAXB; e += CT_THREADS) {
      const int c = e % CT_MAXB;
      rowbuf[e] = (e < CT_MAXB && c < b) ? G[c] : 0.0;
    }
    __syncthreads();
    for (int k = 0; k < b; ++k) {
      const double* rk = rowbuf + (k & 1) * CT_MAXB;
      const double piv = rk[k];
      const double ipiv = piv > 0.0 ? 1.0 / piv : 1.0;
      double gi[NA], gj[NA];
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        const int i = ty + 16 * a, j = tx + 16 * a;
        const double ri = rk[i], rj = rk[j];
        gi[a] = i > k ? ri * ipiv : 0.0;
        gj[a] = j > k ? rj : 0.0;
      }
      // unpredicated: gi / gj are 0 outside the trailing block, where the FMA
      // leaves v unchanged; groups left of the diagonal (c < a) hold only
      // lower-triangle elements, which are never read
#pragma unroll
      for (int a = 0; a < NA; ++a)
#pragma unroll
        for (int c = a; c < NA; ++c) v[a][c] = fma(-gi[a], gj[c], v[a][c]);
      // the owners of row k+1 (one half-warp) publish it; a switch keeps the
      // register array statically indexed
      const int k1 = k + 1;
      if (k1 < b && ty == (k1 & 15)) {
        double* out = rowbuf + (k1 & 1) * CT_MAXB;
        auto publish = [&](const double(&row)[NA], int a0) {
#pragma unroll
          for (int c = 0; c < NA; ++c) {
            const int j = tx + 16 * c;
            if (c >= a0 && j >= k1 && j < b) out[j] = row[c];
          }
        };
        switch (k1 >> 4) {
          case 0: publish(v[0], 0); break;
          case 1: publish(v[1], 1); break;
          case 2: publish(v[2], 2); break;
          case 3: publish(v[3], 3); break;
          case 4: publish(v[4], 4); break;
          case 5: publish(v[5], 5); break;
          default: publish(v[6], 6); break;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int c = 0; c < NA; ++c) {
        const int i = ty + 16 * a, j = tx + 16 * c;
        if (j >= i && j < b) G[i * b + j] = v[a][c];
      }
    __syncthreads();
  }
  for (int k = tid; k < b; k += CT_THREADS) {
    const double piv = G[k * b + k];
    if (!(piv > 0.0)) bad = 1;
    rinv[k] = piv > 0.0 ? 1.0 / sqrt(piv) : 1.0;
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += CT_THREADS) {
    const int i = e / b, j = e - i * b;
    if (j > i) G[e] *= rinv[i];
  }
  __syncthreads();
  // x R = q: x_j = q_j / R_jj, then q_l -= x_j R_jl (l > j); a warp per row,
  // lanes over l
  for (int rr = wy; rr < CT_ROWS; rr += nwy) {
    double* q = qs + rr * (b + 1);
    for (int j = 0; j < b; ++j) {
      const double xj = q[j] * rinv[j];
      __syncwarp();
      if (lane == 0) q[j] = xj;
      for (int l = j + 1 + lane; l < b; l += 32) q[l] = fma(-xj, G[j * b + l], q[l]);
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < CT_ROWS * b; e += CT_THREADS) {
    const int rr = e / b, c = e % b;
    if (r0 + rr < rows) Q[(r0 + rr) * b + c] = qs[rr * (b + 1) + c];
  }
  if (blockIdx.x == 0 && tid == 0) *info = bad;
}

// Q (rows x b) <- orth(Q) by shifted CholeskyQR3.  passes = 2 (shifted, then
// plain) already gives a well-conditioned basis of the same span (orthogonal
// to ~1e-2 at worst, at 1e-16 for moderate condition numbers): enough between
// Rayleigh-Ritz steps, where only the span is carried forward.
static void cholqr2(adg_ctx* ctx, double* Q, int64_t rows, int b, int passes = 3) {
  const bool fused = b <= CT_MAXB;
  DevBuf<double> G((size_t)b * b, ctx->stream), Rinv((size_t)b, ctx->stream);
  DevBuf<GridBarrier> gb(fused ? 0 : 1, ctx->stream);
  DevBuf<int> info(1, ctx->stream);
  info.zero();
  const size_t ct_smem = sizeof(double) * ((size_t)b * b + (size_t)CT_ROWS * (b + 1) + b);
  for (int pass = 0; pass < passes; ++pass) {
    dgemm(ctx, true, false, b, b, rows, 1.0, Q, b, Q, b, 0.0, G.ptr, b);
    // shifted CholeskyQR3: the first pass adds 11 (rows b + b(b+1)) u max(diag)
    const double coef =
        pass == 0 ? 11.0 * ((double)rows * b + (double)b * (b + 1)) * std::ldexp(1.0, -53) : 0.0;
    if (fused) {
      ADG_CUDA(cudaFuncSetAttribute(chol_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ct_smem));
      chol_trsm_kernel<<<(unsigned)((rows + CT_ROWS - 1) / CT_ROWS), CT_THREADS, ct_smem, ctx->stream>>>(
          G.ptr, b, coef, Q, rows, info.ptr);
      after_launch(ctx);
      continue;
    }
    // large b: the factorisation and the solve over the whole grid (cooperative)
    gb.zero();
    int per_sm = 0;
    ADG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chol_trsm_grid_kernel, JG_THREADS, 0));
    ADG_REQUIRE(per_sm >= 1, "cholqr2: grid Cholesky cannot be resident");
    double* gp = G.ptr;
    double* rp = Rinv.ptr;
    int* ip = info.ptr;
    GridBarrier* gbp = gb.ptr;
    int bb = b;
    double cc = coef;
    double* qp = Q;
    int64_t rr = rows;
    void* args[] = {&gp, &bb, &cc, &qp, &rr, &rp, &ip, &gbp};
    ADG_CUDA(cudaLaunchCooperativeKernel((const void*)chol_trsm_grid_kernel, dim3((unsigned)ctx->num_sms),
                                         dim3(JG_THREADS), args, 0, ctx->stream));
    after_launch(ctx);
    if (std::getenv("ADG_CHOLQR_CHECK")) {  // debugging aid
      std::vector<double> hq((size_t)rows * b), hg((size_t)b * b), hr((size_t)b);
      int hinfo = 0;
      ADG_CUDA(cudaMemcpyAsync(hq.data(), Q, hq.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
      ADG_CUDA(cudaMemcpyAsync(hg.data(), G.ptr, hg.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
      ADG_CUDA(cudaMemcpyAsync(hr.data(), Rinv.ptr, hr.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
      ADG_CUDA(cudaMemcpyAsync(&hinfo, info.ptr, 4, cudaMemcpyDeviceToHost, ctx->stream));
      ADG_CUDA(cudaStreamSynchronize(ctx->stream));
      int nq = 0, ng = 0;
      double rmax = 0, rmin = 1e300, qmax = 0;
      for (double v : hq) { nq += std::isnan(v); qmax = std::max(qmax, std::fabs(v)); }
      for (double v : hg) ng += std::isnan(v);
      for (double v : hr) { rmax = std::max(rmax, v); rmin = std::min(rmin, v); }
      std::fprintf(stderr, "[cholqr] b=%d pass=%d info=%d nanQ=%d nanG=%d |Q|max=%.3g rinv[%.3g, %.3g] shiftcoef=%.3g\n",
                   b, pass, hinfo, nq, ng, qmax, rmin, rmax, coef);
    }
  }
}

// ------------------------------------------------------- misc kernels
template <typename T>
__global__ void finite_kernel(const T* __restrict__ X, int64_t count, int* __restrict__ bad) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(to_f64(X[t]))) {
      *bad = 1;
      return;
    }
}

void require_finite(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t count, const char* op) {
  DevBuf<int> bad(1, ctx->stream);
  bad.zero();
  ADG_DISPATCH_DTYPE(dt, T, {
    finite_kernel<T><<<blocks_for(count, 256, 8 * ctx->num_sms), 256, 0, ctx->stream>>>(
        (const T*)X, count, bad.ptr);
  });
  after_launch(ctx);
  int h = 0;
  ADG_CUDA(cudaMemcpyAsync(&h, bad.ptr, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  ADG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h) fail(ADG_ENUMERIC, std::string(op) + ": input contains non-finite values");
}

// basis row k = sign-normalised column k of V (d x ncols): first max-|.| entry > 0
// (proj/src/spectral.cpp:21-27).  One CTA per row.
__global__ void sign_rows_kernel(const double* __restrict__ V, int64_t d, int64_t ncols,
                                 double* __restrict__ basis) {
  const int64_t k = blockIdx.x;
  __shared__ double wv[32];
  __shared__ int64_t wi[32];
  double best = -1.0;
  int64_t bi = INT64_MAX;
  for (int64_t t = threadIdx.x; t < d; t += blockDim.x) {
    const double a = fabs(V[t * ncols + k]);
    if (a > best) {
      best = a;
      bi = t;
    }
  }
  for (int s = 16; s; s >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, s);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, s);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    wv[threadIdx.x >> 5] = best;
    wi[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  __shared__ double sign;
  if (threadIdx.x == 0) {
    double b = -1.0;
    int64_t ii = INT64_MAX;
    for (unsigned w = 0; w < blockDim.x / 32; ++w)
      if (wv[w] > b || (wv[w] == b && wi[w] < ii)) {
        b = wv[w];
        ii = wi[w];
      }
    sign = (ii < d && V[ii * ncols + k] < 0.0) ? -1.0 : 1.0;
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < d; t += blockDim.x) basis[k * d + t] = sign * V[t * ncols + k];
}

// column norms of M (rows x cols) -> out[cols]
__global__ void col_norms_kernel(const double* __restrict__ M, int64_t rows, int64_t cols,
                                 double* __restrict__ out) {
  const int64_t c = blockIdx.x;
  double acc = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    const double v = M[r * cols + c];
    acc = fma(v, v, acc);
  }
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  __shared__ double w[32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (unsigned k = 0; k < blockDim.x / 32; ++k) t += w[k];
    out[c] = sqrt(t);
  }
}

// residual norms ||Z_k - theta_k Y_k|| for k < cols
__global__ void ritz_resid_kernel(const double* __restrict__ Z, const double* __restrict__ Y,
                                  const double* __restrict__ theta, int64_t rows, int64_t ld,
                                  double* __restrict__ out) {
  const int64_t c = blockIdx.x;
  const double th = theta[c];
  double acc = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    const double v = Z[r * ld + c] - th * Y[r * ld + c];
    acc = fma(v, v, acc);
  }
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  __shared__ double w[32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (unsigned k = 0; k < blockDim.x / 32; ++k) t += w[k];
    out[c] = sqrt(t);
  }
}

// centre-and-widen X (n x d) into fp64 (used for one-sided singular values).
template <typename T>
__global__ void widen_center_kernel(const T* __restrict__ X, int64_t n, int64_t d,
                                    const double* __restrict__ mean, double* __restrict__ out) {
  const int64_t total = n * d;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = to_f64(X[t]) - (mean ? mean[t % d] : 0.0);
}

__global__ void sqrt_clamp_kernel(const double* __restrict__ in, int64_t n, double* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = in[t] > 0.0 ? sqrt(in[t]) : 0.0;
}

// Y = M diag(f(vals)) : scale column c of M (rows x cols) by w[c]
__global__ void scale_cols_kernel(double* __restrict__ M, int64_t rows, int64_t cols,
                                  const double* __restrict__ w) {
  const int64_t total = rows * cols;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    M[t] *= w[t % cols];
}

// w[c] = vals[c] > thr ? vals[c]^power : 0   (pseudo-inverse powers)
__global__ void pinv_pow_kernel(const double* __restrict__ vals, int64_t k, double thr, double power,
                                double* __restrict__ w) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < k; t += (int64_t)gridDim.x * blockDim.x)
    w[t] = vals[t] > thr ? pow(vals[t], power) : 0.0;
}

// out = C + delta I (d x d)
__global__ void shift_diag_kernel(const double* __restrict__ C, int64_t d, double delta,
                                  double* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < d * d;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = C[t] + (t / d == t % d ? delta : 0.0);
}

// ------------------------------------------- top eigenvectors of the Gram
// C (d x d, symmetric PSD) -> V (d x want) columns = top eigenvectors, vals.
static void top_eigvecs(adg_ctx* ctx, const double* C, int64_t d, int64_t want, Eig& out) {
  const int64_t b0 = 2 * want + 32;
  // small d, or a block of a quarter of d or more: one Jacobi of the whole
  // Gram (the grid kernel for d > 128; C3: 84 ms, where 232- / 332-column
  // blocks iterate for 205 / 373 ms).  Large blocks can also exceed the
  // Gram's numerical rank (C3 has ~384 constant pixels), where CholeskyQR has
  // no full-rank block to orthonormalise.
  if (d <= 384 || 4 * b0 >= d) {
    sym_eig(ctx, C, (int)d, (int)want, out);
    return;
  }
  const int b = (int)std::min<int64_t>(d, (b0 + 1) / 2 * 2);
  cudaStream_t st = ctx->stream;
  DevBuf<double> Q((size_t)d * b, st), W((size_t)d * b, st), H((size_t)b * b, st),
      Z((size_t)d * b, st), Y((size_t)d * b, st), res((size_t)want, st);
  // deterministic start: fixed-seed Gaussian block, orthonormalised
  normal_device(ctx, 0x5EEDADA61017ULL, d * b, Q.ptr);
  cholqr2(ctx, Q.ptr, d, b);
  const int max_iter = 3000;
  const double tol = 1e-13;
  // A residual that stops halving between Rayleigh-Ritz steps has reached the
  // attainable fp64 floor only once it is this small; above it, slow decay is
  // slow convergence (a flat spectrum around index `want`), never a stop.
  const double floor_rel = 1e-9;
  // iterations the shifted subspace iteration may take before the whole-Gram
  // Jacobi is cheaper and certain (it is exact whatever the spectral gap)
  const int budget = 1200;
  double prev = 1e300;
  int stall = 0, flat = 0;
  bool converged = false;
  // Rayleigh-Ritz (a b x b Jacobi, ~1.8 ms at b = 82) runs at iteration 8,
  // then where the measured geometric decay of the Ritz residual predicts
  // convergence (with a 15 % + 2 margin; a short prediction costs one more
  // Rayleigh-Ritz, a long one a few ~0.15 ms plain iterations)
  //
  // Plain iterations after the second Rayleigh-Ritz step power C - sigma I:
  // the measured per-iteration decay rho ~ lambda_{b+1} / lambda_want gives
  // lambda_{b+1} ~ rho theta_want, and sigma = lambda_{b+1} / 2 centres the
  // unwanted spectrum [0, lambda_{b+1}] on zero (the optimal shift for a PSD
  // Gram), so the rate drops from rho to (rho/2) / (1 - rho/2) (C3: 0.63 ->
  // 0.46).  Same eigenvectors; Rayleigh-Ritz steps use C itself.
  int next_rr = 8, last_rr = 0, n_rr = 0;
  double last_rel = -1.0, sigma = 0.0;
  DevBuf<double> Cs;
  const double* Cit = C;
  Eig e;
  for (int it = 1; it <= max_iter; ++it) {
    const bool rr_step = it == next_rr || it == max_iter;
    dgemm(ctx, false, false, d, b, d, 1.0, rr_step ? C : Cit, d, Q.ptr, b, 0.0, W.ptr, b);  // W = C Q
    if (!rr_step) {
      // plain orthogonal iteration: only the span is carried to the next
      // Rayleigh-Ritz step, so two CholeskyQR passes suffice here
      ADG_CUDA(cudaMemcpyAsync(Q.ptr, W.ptr, sizeof(double) * d * b, cudaMemcpyDeviceToDevice, st));
      cholqr2(ctx, Q.ptr, d, b, 2);
      continue;
    }
    ++n_rr;
    dgemm(ctx, true, false, b, b, d, 1.0, Q.ptr, b, W.ptr, b, 0.0, H.ptr, b);  // H = Q^T C Q
    sym_eig(ctx, H.ptr, b, b, e);                                              // Rayleigh-Ritz
    dgemm(ctx, false, false, d, b, b, 1.0, W.ptr, b, e.vecs.ptr, b, 0.0, Z.ptr, b);  // Z = C Y
    {
      dgemm(ctx, false, false, d, b, b, 1.0, Q.ptr, b, e.vecs.ptr, b, 0.0, Y.ptr, b);  // Y = Q U
      ritz_resid_kernel<<<(unsigned)want, 256, 0, st>>>(Z.ptr, Y.ptr, e.vals.ptr, d, b, res.ptr);
      after_launch(ctx);
      std::vector<double> hr((size_t)want), hth((size_t)want);
      ADG_CUDA(cudaMemcpyAsync(hr.data(), res.ptr, sizeof(double) * want, cudaMemcpyDeviceToHost, st));
      ADG_CUDA(cudaMemcpyAsync(hth.data(), e.vals.ptr, sizeof(double) * want, cudaMemcpyDeviceToHost, st));
      ADG_CUDA(cudaStreamSynchronize(st));
      const double th0 = hth[0];
      double worst = 0.0;
      for (double v : hr) worst = std::max(worst, v);
      const double rel = th0 > 0.0 ? worst / th0 : 0.0;
      if (rel >= 0.5 * prev && rel < floor_rel)
        ++stall;  // at the fp64 floor once this persists
      else
        stall = 0;
      flat = (last_rel > 0.0 && rel >= last_rel) ? flat + 1 : 0;  // no progress at all
      prev = std::min(prev, rel);
      converged = rel <= tol || stall >= 4;
      const bool give_up = !converged && (it == max_iter || flat >= 3);
      if (converged || give_up) {
        if (std::getenv("ADG_FIT_PROFILE"))
          std::fprintf(stderr, "[fit] subspace iteration: d=%lld b=%d iterations=%d rayleigh_ritz=%d residual=%.3g shift=%.4g%s\n",
                       (long long)d, b, it, n_rr, rel, sigma, converged ? "" : " (not converging: whole-Gram Jacobi)");
        break;
      }
      int step = 8;
      if (last_rel > 0.0 && rel > 0.0 && rel < last_rel) {
        double per_it = std::log(rel / last_rel) / (double)(it - last_rr);  // < 0
        const double rho = std::exp(per_it);
        const double th_want = hth[(size_t)want - 1];
        if (sigma == 0.0 && rho < 0.98 && th_want > 0.0 && !std::getenv("ADG_NO_SHIFT")) {
          sigma = 0.5 * rho * th_want;
          Cs.alloc((size_t)d * d, st);
          shift_diag_kernel<<<blocks_for(d * d, 256, 4 * ctx->num_sms), 256, 0, st>>>(C, d, -sigma, Cs.ptr);
          after_launch(ctx);
          Cit = Cs.ptr;
          per_it = std::log(0.5 * rho / (1.0 - 0.5 * rho));  // predicted shifted rate
        }
        const double need = std::log(tol / rel) / per_it;
        if (rel > floor_rel && (double)it + need > (double)budget) {
          // too flat a spectrum for the block: converging would take longer
          // than the direct solve
          if (std::getenv("ADG_FIT_PROFILE"))
            std::fprintf(stderr, "[fit] subspace iteration: d=%lld b=%d predicted %.0f more iterations "
                         "at rate %.4f: whole-Gram Jacobi\n", (long long)d, b, need, std::exp(per_it));
          break;
        }
        step = (int)std::min(64.0, std::max(4.0, std::ceil(1.15 * need) + 2.0));
      }
      last_rel = rel;
      last_rr = it;
      next_rr = it + step;
    }
    ADG_CUDA(cudaMemcpyAsync(Q.ptr, Z.ptr, sizeof(double) * d * b, cudaMemcpyDeviceToDevice, st));
    cholqr2(ctx, Q.ptr, d, b);
  }
  if (!converged) {
    // exact whatever the spectrum (the reference's BDCSVD is, spectral.cpp:52)
    sym_eig(ctx, C, (int)d, (int)want, out);
    return;
  }
  // keep the first `want` Ritz vectors (columns of Y, already sorted)
  out.vals.alloc((size_t)want, st);
  out.vecs.alloc((size_t)d * want, st);
  ADG_CUDA(cudaMemcpy2DAsync(out.vecs.ptr, sizeof(double) * want, Y.ptr, sizeof(double) * b,
                             sizeof(double) * want, d, cudaMemcpyDeviceToDevice, st));
  ADG_CUDA(cudaMemcpyAsync(out.vals.ptr, e.vals.ptr, sizeof(double) * want, cudaMemcpyDeviceToDevice, st));
}

// Top-s rows of the centred Gram C (d x d): sign-normalised basis; the Ritz
// vectors (d x want) are left in `e` for the one-sided singular values.
static void spectral_from_gram(adg_ctx* ctx, const double* C, int64_t d, int64_t s, int64_t want,
                               double* basis_out, Eig& e) {
  top_eigvecs(ctx, C, d, want, e);
  sign_rows_kernel<<<(unsigned)s, 256, 0, ctx->stream>>>(e.vecs.ptr, d, want, basis_out);
  after_launch(ctx);
}

void spectral_exact_gram(adg_ctx* ctx, const double* C, int64_t d, int64_t s, double* basis_out) {
  Eig e;
  spectral_from_gram(ctx, C, d, s, s, basis_out, e);
}

void spectral_exact(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d,
                    const double* mean, int64_t s, double* basis_out, double* sigma_out,
                    int64_t n_sigma, const char* opname) {
  const bool prof = std::getenv("ADG_FIT_PROFILE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!prof) return;
    cudaStreamSynchronize(ctx->stream);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[fit] %-10s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  };
  require_finite(ctx, X, dt, n * d, opname);
  mark("finite");
  cudaStream_t st = ctx->stream;
  DevBuf<double> C((size_t)d * d, st);
  gram_f64(ctx, X, dt, n, d, mean, C.ptr);
  mark("gram");
  const int64_t want = std::max<int64_t>(s, n_sigma);
  Eig e;
  spectral_from_gram(ctx, C.ptr, d, s, want, basis_out, e);
  mark("eig");
  if (sigma_out && n_sigma > 0) {
    // one-sided: sigma_k = || Xc v_k ||
    DevBuf<double> Xc((size_t)(n * d), st), XV((size_t)(n * want), st);
    ADG_DISPATCH_DTYPE(dt, T, {
      widen_center_kernel<T><<<blocks_for(n * d, 256, 8 * ctx->num_sms), 256, 0, st>>>(
          (const T*)X, n, d, mean, Xc.ptr);
    });
    after_launch(ctx);
    dgemm(ctx, false, false, n, want, d, 1.0, Xc.ptr, d, e.vecs.ptr, want, 0.0, XV.ptr, want);
    DevBuf<double> norms((size_t)want, st);
    col_norms_kernel<<<(unsigned)want, 256, 0, st>>>(XV.ptr, n, want, norms.ptr);
    after_launch(ctx);
    ADG_CUDA(cudaMemcpyAsync(sigma_out, norms.ptr, sizeof(double) * n_sigma, cudaMemcpyDeviceToDevice, st));
  }
}

void spectral_randomized(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d,
                         const double* mean, int64_t s, int64_t oversampling, int power_iters,
                         uint64_t seed, double* basis_out, double* sigma_out) {
  require_finite(ctx, X, dt, n * d, "randomized_top_svd");
  DevBuf<double> C((size_t)d * d, ctx->stream);
  gram_f64(ctx, X, dt, n, d, mean, C.ptr);
  spectral_randomized_gram(ctx, C.ptr, d, s, oversampling, power_iters, seed, basis_out, sigma_out);
}

void spectral_randomized_gram(adg_ctx* ctx, const double* C_in, int64_t d, int64_t s,
                              int64_t oversampling, int power_iters, uint64_t seed,
                              double* basis_out, double* sigma_out) {
  cudaStream_t st = ctx->stream;
  const int64_t w = s + oversampling;
  const double* C = C_in;
  // Omega: d x w, SeededRng(seed).normal() row-major (spectral.cpp:79-82)
  DevBuf<double> Z((size_t)d * w, st), K((size_t)d * w, st);
  normal_device(ctx, seed, d * w, Z.ptr);
  for (int q = 0; q < power_iters; ++q) {
    // span(X^T X Z): one power pass of the reference's range finder
    cholqr2(ctx, Z.ptr, d, (int)w);
    dgemm(ctx, false, false, d, w, d, 1.0, C, d, Z.ptr, w, 0.0, K.ptr, w);
    ADG_CUDA(cudaMemcpyAsync(Z.ptr, K.ptr, sizeof(double) * d * w, cudaMemcpyDeviceToDevice, st));
  }
  cholqr2(ctx, Z.ptr, d, (int)w);
  // K = C Z, G = Z^T C Z; B^T B = K G^+ K^T = F F^T with F = K G^{-1/2}
  dgemm(ctx, false, false, d, w, d, 1.0, C, d, Z.ptr, w, 0.0, K.ptr, w);
  DevBuf<double> G((size_t)w * w, st);
  dgemm(ctx, true, false, w, w, d, 1.0, Z.ptr, w, K.ptr, w, 0.0, G.ptr, w);
  Eig eg;
  sym_eig(ctx, G.ptr, (int)w, (int)w, eg);
  double gmax = 0.0;
  ADG_CUDA(cudaMemcpyAsync(&gmax, eg.vals.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
  ADG_CUDA(cudaStreamSynchronize(st));
  DevBuf<double> wv((size_t)w, st), Gih((size_t)w * w, st), U2((size_t)w * w, st),
      F((size_t)d * w, st);
  const double thr = std::max(gmax, 0.0) * (double)w * 1e-15;
  pinv_pow_kernel<<<1, 256, 0, st>>>(eg.vals.ptr, w, thr, -0.5, wv.ptr);
  after_launch(ctx);
  // G^{-1/2} = U diag(wv) U^T
  ADG_CUDA(cudaMemcpyAsync(U2.ptr, eg.vecs.ptr, sizeof(double) * w * w, cudaMemcpyDeviceToDevice, st));
  scale_cols_kernel<<<blocks_for(w * w, 256), 256, 0, st>>>(U2.ptr, w, w, wv.ptr);
  after_launch(ctx);
  dgemm(ctx, false, true, w, w, w, 1.0, U2.ptr, w, eg.vecs.ptr, w, 0.0, Gih.ptr, w);
  dgemm(ctx, false, false, d, w, w, 1.0, K.ptr, w, Gih.ptr, w, 0.0, F.ptr, w);
  // T = F^T F = Ut S^2 Ut^T; top-s left singular vectors of F: F Ut S^-1
  DevBuf<double> T((size_t)w * w, st);
  dgemm(ctx, true, false, w, w, d, 1.0, F.ptr, w, F.ptr, w, 0.0, T.ptr, w);
  Eig et;
  sym_eig(ctx, T.ptr, (int)w, (int)s, et);
  DevBuf<double> sig((size_t)s, st), inv((size_t)s, st), V((size_t)d * s, st);
  sqrt_clamp_kernel<<<1, 256, 0, st>>>(et.vals.ptr, s, sig.ptr);
  after_launch(ctx);
  double tmax = 0.0;
  ADG_CUDA(cudaMemcpyAsync(&tmax, et.vals.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
  ADG_CUDA(cudaStreamSynchronize(st));
  pinv_pow_kernel<<<1, 256, 0, st>>>(et.vals.ptr, s, std::max(tmax, 0.0) * 1e-28, -0.5, inv.ptr);
  after_launch(ctx);
  dgemm(ctx, false, false, d, s, w, 1.0, F.ptr, w, et.vecs.ptr, s, 0.0, V.ptr, s);
  scale_cols_kernel<<<blocks_for(d * s, 256), 256, 0, st>>>(V.ptr, d, s, inv.ptr);
  after_launch(ctx);
  sign_rows_kernel<<<(unsigned)s, 256, 0, st>>>(V.ptr, d, s, basis_out);
  after_launch(ctx);
  if (sigma_out)
    ADG_CUDA(cudaMemcpyAsync(sigma_out, sig.ptr, sizeof(double) * s, cudaMemcpyDeviceToDevice, st));
}

}  // namespace adg
