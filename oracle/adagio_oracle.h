/*
 * adagio_oracle.h -- CPU restatement of the ADAgIO reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 product path (paper_1609_05388_b200/libadg.so).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product never links, calls or falls back to it.
 *
 * Every function restates the reference algorithm in plain C (fp64, the
 * reference's precision) and cites the reference file:line it follows
 * (paths relative to the reference checkout, proj/...).  The reference itself
 * needs Eigen >= 3.3 (proj/CMakeLists.txt:12), which is absent from this
 * image, so it is unbuildable here; the header-only proj/include/adagio/rng.hpp
 * IS compiled from the reference sources by oracle/Makefile (target ref) and
 * pins this restatement's RNG bit-for-bit (tests/golden/rng_golden.json).
 * The evaluate / jl / transform / center restatements are pinned against the
 * reference's own known-answer tests (proj/tests/test_*.cpp), restated in
 * tests/test_oracle.py.
 */
#ifndef ADAGIO_ORACLE_H
#define ADAGIO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/include/adagio/rng.hpp:11-44 */
uint64_t or_mix64(uint64_t x);
uint64_t or_fnv1a64(const char* bytes, int64_t len);
uint64_t or_derive_seed(uint64_t seed, const char* purpose);
uint64_t or_hash_position(uint64_t seed, uint64_t i, uint64_t j);
double or_rademacher_sign(uint64_t seed, uint64_t i, uint64_t j);

/* SeededRng, proj/include/adagio/rng.hpp:49-91: fill helpers. */
void or_rng_u64(uint64_t seed, int64_t count, uint64_t* out);
void or_rng_below(uint64_t seed, uint64_t bound, int64_t count, uint64_t* out);
void or_rng_normal(uint64_t seed, int64_t count, double* out);

/* proj/src/jl.cpp:13-36 (k x d row-major) and jl.cpp:38-50. */
int or_sample_jl(int64_t k, int64_t d, uint64_t seed, double* out);
int64_t or_jl_dimension(int64_t n_points, double epsilon, double gamma);

/* proj/src/dataset.cpp:209-216: mean[d]; centered may be NULL. */
void or_center(const double* X, int64_t n, int64_t d, double* mean, double* centered);

/* proj/src/embed.cpp:143-181: rows of X (n x d) -> out (n x (s+k)). */
void or_transform_all(const double* mean, const double* P, int64_t s, const double* S,
                      int64_t k, int64_t d, const double* X, int64_t n, double* out,
                      int threads);

/* proj/include/adagio/distortion.hpp:32-42 plus the argmax extension
 * (lowest linear pair index among exact ties). */
typedef struct {
  double max_distortion;
  double mean_distortion;
  uint64_t n_pairs_evaluated;
  uint64_t n_zero_distance_pairs;
  uint64_t argmax_i;  /* UINT64_MAX when nothing was evaluated */
  uint64_t argmax_j;
  int32_t hist_bins;
  int32_t sampled;
  double hist_max;
  uint64_t sample_seed;
} or_report;

/* proj/src/distortion.cpp:113-192.  hist must hold hist_bins+1 counts.
 * edge_band > 0 additionally counts, per edge e = 1..hist_bins (edge value
 * e*hist_max/hist_bins), the pairs whose exact value lies within edge_band of
 * it (edge_near[e-1]) and within 10*edge_band (edge_near[hist_bins+e-1]);
 * edge_near holds 2*hist_bins counts; used by tests to bound "exact away from
 * bin edges".
 * edge_near may be NULL.  row_begin/row_end restrict all-pairs mode to pairs
 * whose first index lies in [row_begin,row_end) (bounded CPU-baseline
 * samples); pass 0 / n for the full job.  Returns 0 or -1 on bad arguments. */
int or_evaluate(const double* orig, int64_t n, int64_t d, const double* emb, int64_t n_emb,
                int64_t r, int all_pairs, uint64_t m, uint64_t sample_seed, int hist_bins,
                double hist_max, uint64_t pairs_per_block, int threads, or_report* rep,
                uint64_t* hist, double edge_band, uint64_t* edge_near, int64_t row_begin,
                int64_t row_end);

/* Same, fp32 inputs widened exactly to fp64 on the fly (bench CPU baseline
 * on the same fp32 files the GPU reads). */
int or_evaluate_f32(const float* orig, int64_t n, int64_t d, const float* emb, int64_t r,
                    int hist_bins, double hist_max, int threads, or_report* rep, uint64_t* hist,
                    int64_t row_begin, int64_t row_end);

/* TEST INFRASTRUCTURE (not a reference function): per-edge counts of the
 * pairs whose exact value lies within the GPU SCREEN's rigorous per-pair
 * error bound t = rel_eps (sn/o + sm/e)(1 + v) of a bin edge (out[0, bins))
 * and within frac * t (out[bins, 2 bins)); nx / ny are the rows' squared
 * norms after the screen's centring shift.  fp32 clouds, all pairs. */
int or_edge_band_counts(const float* x, const float* y, int64_t n, int64_t d, int64_t r,
                        const double* nx, const double* ny, double rel_eps, double frac,
                        int hist_bins, double hist_max, int threads, uint64_t* out);

/* Sampled mode (distortion.cpp:90-103, :151-154) on fp32 clouds, widened
 * exactly to fp64 on the fly (C4 / C5 parity without an fp64 copy). */
int or_evaluate_f32_sampled(const float* orig, int64_t n, int64_t d, const float* emb, int64_t r,
                            uint64_t m, uint64_t sample_seed, int hist_bins, double hist_max,
                            int threads, or_report* rep, uint64_t* hist);

/* proj/src/distortion.cpp:46-57 */
void or_decode_pair(uint64_t p, uint64_t n, uint64_t* i, uint64_t* j);
/* proj/src/distortion.cpp:90-103 (sorted output, m entries). */
int or_sample_pair_indices(uint64_t total, uint64_t m, uint64_t seed, uint64_t* out);
/* proj/src/distortion.cpp:107-111; returns -1.0 for coincident points. */
double or_pair_distortion(const double* x, const double* y, const double* fx, const double* fy,
                          int64_t d, int64_t r);

/* proj/tests/test_util.hpp:57-84: independent naive double loop, long-double mean. */
void or_naive_distortion(const double* orig, int64_t n, int64_t d, const double* emb, int64_t r,
                         double* max_out, double* mean_out, uint64_t* evaluated,
                         uint64_t* zero_pairs);

#ifdef __cplusplus
}
#endif
#endif
