// adg_spectral.cuh -- interfaces of adg_spectral.cu
#pragma once
#include "adg_embed.cuh"

namespace adg {

// proj/src/spectral.cpp:42-62.  X (n x d, device), centred by mean (device,
// nullable = as given).  basis_out (s x d, device) sign-normalised rows;
// sigma_out (device, nullable) the n_sigma largest singular values.  When
// s > min(n, d) the rows are the top-s eigenvectors of the full Gram
// (proj/src/embed.cpp:46-55 full-V branch).
void spectral_exact(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d,
                    const double* mean, int64_t s, double* basis_out, double* sigma_out,
                    int64_t n_sigma, const char* opname);

// proj/src/spectral.cpp:64-101 (Halko), via the Gram.
void spectral_randomized(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d,
                         const double* mean, int64_t s, int64_t oversampling, int power_iters,
                         uint64_t seed, double* basis_out, double* sigma_out);

// The same solves on a precomputed centred Gram C (d x d, device): the
// row-sharded fit all-reduces the per-shard Grams and calls these on every
// rank.
void spectral_exact_gram(adg_ctx* ctx, const double* C, int64_t d, int64_t s, double* basis_out);
void spectral_randomized_gram(adg_ctx* ctx, const double* C, int64_t d, int64_t s,
                              int64_t oversampling, int power_iters, uint64_t seed,
                              double* basis_out, double* sigma_out);
// ADG_ENUMERIC "<op>: input contains non-finite values" unless all finite.
void require_finite(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t count, const char* op);

// fp64 building blocks (row-major).  C = alpha * op(A) op(B) + beta * C.
void dgemm(adg_ctx* ctx, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
           const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
           int64_t ldc);
// Gram of the centred rows [0, n): G (d x d, full symmetric), deterministic.
void gram_f64(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d,
              const double* mean, double* G);

}  // namespace adg
