/*
 * adg.h -- C ABI of the B200-native ADAgIO hot path (libadg.so).
 *
 * Drop-in boundary for the reference's C++ free-function API
 * (proj/include/adagio/{embed,distortion,spectral,jl,dataset}.hpp).  Plain
 * pointers and sizes only; no CUDA, Eigen or torch types.  Every data pointer
 * may be HOST or DEVICE memory (detected with cudaPointerGetAttributes): host
 * buffers are staged through the context's stream, device buffers are used in
 * place, so fit -> transform -> evaluate can stay resident in HBM.
 *
 * Matrices are row-major, one point per row, exactly like the reference's
 * Matrix = Eigen::Matrix<double, Dynamic, Dynamic, RowMajor>
 * (proj/include/adagio/point_cloud.hpp:12).  The reference is fp64-only; here
 * the input dtype is chosen per call (ADG_F64 / ADG_F32 / ADG_BF16) and model
 * outputs (mean, basis, sketch) are always fp64 like the reference's.
 *
 * Errors: every call returns an adg_status; adg_last_error() holds the message
 * of the last failure on the calling thread, with the reference's message
 * prefixes ("evaluate: cloud sizes differ (...)", "fit: target_dim = ...").
 * Status -> reference exception: ADG_EINVAL -> std::invalid_argument,
 * ADG_ENUMERIC -> adagio::NumericError, ADG_EIO -> adagio::IoError
 * (proj/include/adagio/errors.hpp:10-18); ADG_ECUDA is new (device failure).
 *
 * Every function here runs its arithmetic on the GPU; there is no CPU path.
 */
#ifndef ADG_H
#define ADG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADG_ABI_VERSION 2

typedef enum {
  ADG_OK = 0,
  ADG_EINVAL = 1,   /* std::invalid_argument in the reference */
  ADG_ENUMERIC = 2, /* adagio::NumericError (errors.hpp:16) */
  ADG_EIO = 3,      /* adagio::IoError (errors.hpp:10) */
  ADG_ECUDA = 4,    /* CUDA / device failure (no reference analogue) */
  ADG_ENOMEM = 5,
  ADG_ENCCL = 6     /* a collective of the multi-GPU exchange failed */
} adg_status;

typedef enum { ADG_F64 = 0, ADG_F32 = 1, ADG_BF16 = 2 } adg_dtype;

/* proj/include/adagio/embed.hpp:12 */
typedef enum { ADG_BACKEND_EXACT = 0, ADG_BACKEND_RANDOMIZED = 1 } adg_backend;

/* Distortion engine: AUTO picks EXACT (fp64 direct differences for every
 * pair, the reference's own formula) for small jobs and SCREEN (tcgen05
 * split-fp16 Gram screen + exact fp64 refine of the max band) otherwise. */
/* AUTO: EXACT for n <= 4096 and sampled mode, else SCREEN.  SCREEN: max,
 * argmax, counts exact; a pair is binned from its screened value (exact away
 * from bin edges).  SCREEN_EXACT_HIST: SCREEN, plus every pair whose screened
 * value lies within the edge band of a bin edge binned by its exact fp64
 * value. */
typedef enum {
  ADG_ENGINE_AUTO = 0,
  ADG_ENGINE_EXACT = 1,
  ADG_ENGINE_SCREEN = 2,
  ADG_ENGINE_SCREEN_EXACT_HIST = 3
} adg_engine;

typedef struct adg_ctx adg_ctx;

/* ----------------------------------------------------------------- context */
int adg_abi_version(void);
const char* adg_last_error(void);
/* One context per host thread (or guard it); binds a device and a stream. */
adg_status adg_ctx_create(int device, adg_ctx** out);
adg_status adg_ctx_destroy(adg_ctx* ctx);
/* stream: a cudaStream_t (NULL = the context's own non-blocking stream; pass
   cudaStreamLegacy, (void*)0x1, to order work with the legacy default stream). */
adg_status adg_ctx_set_stream(adg_ctx* ctx, void* stream);
adg_status adg_ctx_synchronize(adg_ctx* ctx);

/* -------------------------------------------------- rng.hpp / jl.cpp / seeds */
/* proj/include/adagio/rng.hpp:30-32 (host scalar; seeds are bookkeeping). */
uint64_t adg_derive_seed(uint64_t seed, const char* purpose);

/* proj/src/jl.cpp:13-36 -> out[k*d] (fp64, row-major): entry (i,j) =
 * (1/sqrt(k)) * rademacher_sign(seed, i, j), bit-exact.  Replaces
 * adagio::sample_jl (proj/include/adagio/jl.hpp:22). */
adg_status adg_sample_jl(adg_ctx* ctx, int64_t k, int64_t d, uint64_t seed, double* out);

/* proj/src/jl.cpp:38-50 (host scalar formula). */
adg_status adg_jl_dimension(int64_t n_points, double epsilon, double gamma, int64_t* out);

/* ------------------------------------------------------------ dataset.cpp */
/* proj/src/dataset.cpp:209-216 -> mean[d] (fp64); centered (n x d, same
 * dtype as X) may be NULL.  Replaces adagio::center (dataset.hpp:36). */
adg_status adg_center(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                      double* mean_out, void* centered_out);

/* ----------------------------------------------------------- spectral.cpp */
/* proj/src/spectral.cpp:42-62: top-s right singular rows of X (n x d, used as
 * given, not centred) -> basis_out[s*d] (fp64, rows sign-normalised so the
 * first max-|.| entry is positive).  sigma_out (may be NULL) receives the
 * n_sigma <= min(n, d) largest singular values, descending.  Replaces
 * adagio::exact_top_svd (spectral.hpp:29). */
adg_status adg_exact_top_svd(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                             int64_t s, double* basis_out, double* sigma_out, int64_t n_sigma);

/* proj/src/spectral.cpp:64-101 (Halko, Gaussian test matrix from
 * SeededRng(seed).normal(), power_iters re-orthonormalised passes) ->
 * basis_out[s*d], sigma_out[s] (approximate).  Replaces
 * adagio::randomized_top_svd (spectral.hpp:35). */
adg_status adg_randomized_top_svd(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n,
                                  int64_t d, int64_t s, int64_t oversampling, int power_iters,
                                  uint64_t seed, double* basis_out, double* sigma_out);

/* -------------------------------------------------------------- embed.cpp */
/* proj/src/embed.cpp:115-141 (AdagioModel fit_with_split): mean_out[d],
 * basis_out[s*d], sketch_out[k*d], all fp64.  The sketch seed is
 * derive_seed(seed, "jl") and the randomized backend uses
 * derive_seed(seed, "spectral") exactly as the reference. */
adg_status adg_fit_with_split(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n,
                              int64_t d, int64_t s, int64_t k, adg_backend backend,
                              uint64_t seed, double* mean_out, double* basis_out,
                              double* sketch_out);

/* Row-sharded fit (no single reference function: it is
 * fit_with_split, proj/src/embed.cpp:115-141, with the column mean
 * (dataset.cpp:211) and the Gram behind exact_top_svd / randomized_top_svd
 * (spectral.cpp:42-101) computed per row shard and all-reduced by the
 * caller).  With one shard the three calls reproduce adg_fit_with_split bit
 * for bit:
 *   sums[d]   = adg_column_sums(shard)            -> all-reduce SUM, mean = sums / n_total
 *   gram[d*d] = adg_gram(shard, mean)              -> all-reduce SUM
 *   basis[s*d], sketch[k*d] = adg_fit_from_gram(gram, n_total, ...) on every rank.
 * adg_gram fails with ADG_ENUMERIC (the reference's NumericError text of the
 * backend's SVD) on a non-finite shard; an empty shard (n = 0) gives zeros. */
adg_status adg_column_sums(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                           double* sums_out);
adg_status adg_gram(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                    const double* mean, adg_backend backend, double* gram_out);
adg_status adg_fit_from_gram(adg_ctx* ctx, const double* gram, int64_t n_total, int64_t d,
                             int64_t s, int64_t k, adg_backend backend, uint64_t seed,
                             double* basis_out, double* sketch_out);

/* proj/src/embed.cpp:105-113: s = floor(r/2), k = r - s. */
adg_status adg_fit(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                   int64_t target_dim, adg_backend backend, uint64_t seed, double* mean_out,
                   double* basis_out, double* sketch_out);

/* proj/src/embed.cpp:143-181 (transform / transform_all): Y[n, s+k] with the
 * first s columns principal coordinates, the last k the sketch of the
 * residual.  out_dtype ADG_F64 or ADG_F32.  fp64 inputs are computed in fp64,
 * fp32/bf16 inputs in fp32 with fp64 model constants. */
adg_status adg_transform_all(adg_ctx* ctx, const double* mean, const double* basis, int64_t s,
                             const double* sketch, int64_t k, int64_t d, const void* X,
                             adg_dtype dtype, int64_t n, void* Y_out, adg_dtype out_dtype);

/* The same transform with the model prepared once (W = [P ; S(I - P^T P)] in
 * the compute type, its tf32 split, the padded mean) for repeated
 * transform_all calls with one model.  input_dtype selects the compute type
 * exactly as adg_transform_all does (ADG_F64 -> fp64; ADG_F32 / ADG_BF16 ->
 * fp32); run accepts inputs of that class only (ADG_EINVAL otherwise).
 * Results are bit-identical to adg_transform_all. */
typedef struct adg_transform_plan adg_transform_plan;
adg_status adg_transform_plan_create(adg_ctx* ctx, const double* mean, const double* basis,
                                     int64_t s, const double* sketch, int64_t k, int64_t d,
                                     adg_dtype input_dtype, adg_transform_plan** out);
adg_status adg_transform_plan_run(adg_transform_plan* plan, const void* X, adg_dtype dtype,
                                  int64_t n, void* Y_out, adg_dtype out_dtype);
adg_status adg_transform_plan_destroy(adg_transform_plan* plan);

/* --------------------------------------------------------- distortion.cpp */
/* proj/include/adagio/distortion.hpp:16-25 */
typedef struct {
  int32_t all_pairs; /* 1 = every unordered pair once */
  int32_t _pad;
  uint64_t m;        /* sampled: number of distinct pairs */
  uint64_t seed;     /* sampled: SeededRng seed for Floyd's algorithm */
} adg_pair_sampling;

/* proj/include/adagio/distortion.hpp:32-42 plus the argmax extension
 * (lowest (i, j) among exact ties; UINT64_MAX when nothing was evaluated). */
typedef struct {
  double max_distortion;
  double mean_distortion;
  uint64_t n_pairs_evaluated;
  uint64_t n_zero_distance_pairs;
  uint64_t argmax_i;
  uint64_t argmax_j;
  int32_t hist_bins;
  int32_t sampled;
  double hist_max;
  uint64_t sample_seed;
  int32_t engine;         /* adg_engine actually used */
  int32_t candidate_rows; /* SCREEN: rows refined exactly for the max */
  double screen_error_bound; /* SCREEN: per-pair |screened - exact| bound used */
  uint64_t edge_pairs;       /* SCREEN: pairs binned by the exact fp64 value because their
                                screened value lay within the edge band of a bin edge */
} adg_report;

/* proj/src/distortion.cpp:113-192 (evaluate).  hist_out receives
 * hist_bins + 1 counts (overflow last).  pairs_per_block is accepted and is
 * results-neutral, as documented at distortion.hpp:47-51. */
adg_status adg_evaluate(adg_ctx* ctx, const void* orig, adg_dtype orig_dtype, int64_t n,
                        int64_t d, const void* emb, adg_dtype emb_dtype, int64_t n_emb,
                        int64_t r, const adg_pair_sampling* mode, int hist_bins,
                        double hist_max, uint64_t pairs_per_block, adg_engine engine,
                        adg_report* report, uint64_t* hist_out);

/* proj/tools/adagio_main.cpp:192-224 (run_distort with --model): embedded =
 * transform_all(model, X) (proj/src/embed.cpp:161-181), then evaluate(X,
 * embedded, mode, hist_bins, hist_max).  Same results as adg_transform_all
 * followed by adg_evaluate on an embedding of dtype y_dtype (ADG_F32/ADG_F64),
 * but X is staged to the device once and the embedding stays in HBM; Y_out
 * (n x (s+k) of y_dtype, host or device, may be NULL) receives it if given. */
adg_status adg_distort_model(adg_ctx* ctx, const double* mean, const double* basis, int64_t s,
                             const double* sketch, int64_t k, int64_t d, const void* X,
                             adg_dtype dtype, int64_t n, const adg_pair_sampling* mode,
                             int hist_bins, double hist_max, adg_engine engine,
                             adg_report* report, uint64_t* hist_out, void* Y_out,
                             adg_dtype y_dtype);

/* proj/src/distortion.cpp:194-196 */
adg_status adg_max_distortion(adg_ctx* ctx, const void* orig, adg_dtype orig_dtype, int64_t n,
                              int64_t d, const void* emb, adg_dtype emb_dtype, int64_t r,
                              double* out);

/* proj/src/distortion.cpp:107-111 (coincident points -> ADG_EINVAL). */
adg_status adg_pair_distortion(adg_ctx* ctx, const double* x, const double* y, int64_t d,
                               const double* fx, const double* fy, int64_t r, double* out);

/* proj/src/distortion.cpp:198-230: output layout (host formatting).  Return
 * the number of bytes needed (excluding NUL); write at most cap bytes. */
size_t adg_report_to_json(const adg_report* report, const uint64_t* hist, char* buf, size_t cap);
size_t adg_histogram_csv(const adg_report* report, const uint64_t* hist, char* buf, size_t cap);

/* ------------------------------------------- sharded evaluation (multi-GPU)
 * SURVEY 8(e).  The SCREEN engine's pair space is a list of 256 x 160 tiles
 * of the upper triangle.  A plan prepares the device operands once; each rank
 * (one per GPU) screens a contiguous tile range (adg_eval_plan_run), the
 * ranks combine their partials with adg_eval_plan_exchange, and every rank
 * finalizes to the identical report -- bit-identical for any GPU count, the
 * GPU analogue of the reference's thread-count invariance
 * (proj/include/adagio/parallel.hpp:8-11).  Partials are device pointers
 * owned by the plan. */
typedef struct adg_eval_plan adg_eval_plan;

/* Collectives of the exchange.  The library calls them in the same order on
 * every rank, on device buffers, with the plan's stream (a cudaStream_t the
 * collective must be ordered on); each returns 0 on success.  Provided by
 * adg_comm_nccl_* (NCCL over NVLink / NVSwitch, loaded at run time) or by the
 * caller (the Python layer binds torch.distributed, NCCL or host-staged gloo). */
typedef enum { ADG_SUM_U64 = 0, ADG_SUM_F64 = 1, ADG_MAX_F32 = 2, ADG_MAX_U64 = 3 } adg_reduce_op;
typedef struct {
  int32_t world;
  int32_t rank;
  void* user;
  /* in place: buf[count] of the op's type, reduced over all ranks */
  int (*all_reduce)(void* user, void* buf, int64_t count, int32_t op, void* stream);
  /* recv[world * bytes] = every rank's send[bytes], in rank order */
  int (*all_gather)(void* user, const void* send, void* recv, int64_t bytes, void* stream);
} adg_collectives;

/* NCCL communicators.  Multi-process (one rank per process): rank 0 draws
 * the id (adg_nccl_unique_id), the caller broadcasts it, every rank calls
 * adg_comm_nccl_create on its own context.  Single process, one rank per
 * listed device: adg_comm_nccl_create_all fills comms[ndev].  ADG_ENCCL if
 * libnccl.so.2 cannot be loaded. */
adg_status adg_nccl_unique_id(uint8_t id_out[128]);
adg_status adg_comm_nccl_create(adg_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128],
                                adg_collectives* out);
adg_status adg_comm_nccl_create_all(int32_t ndev, const int32_t* devices, adg_collectives* comms);
adg_status adg_comm_nccl_destroy(adg_collectives* comm);

typedef struct {
  uint64_t* hist;        /* hist_bins + 1, SUM */
  double* tile_sums;     /* tile_slots * num_tiles, SUM (zero outside the rank's range) */
  float* row_max;        /* n (screened max per first index), MAX */
  float* row_bound;      /* n (screened max + error bound), MAX */
  uint32_t* near_pairs;  /* 2 * near_capacity (i, j) pairs needing exact check */
  uint64_t* near_count;  /* 1 (count may exceed capacity => overflow) */
  int64_t num_tiles;
  int64_t near_capacity;
  int64_t n;
  int32_t hist_bins;
  int32_t tile_slots;    /* partial-sum slots per tile */
} adg_eval_partials;

adg_status adg_eval_plan_create(adg_ctx* ctx, const void* orig, adg_dtype orig_dtype, int64_t n,
                                int64_t d, const void* emb, adg_dtype emb_dtype, int64_t r,
                                int hist_bins, double hist_max, adg_eval_plan** out);
adg_status adg_eval_plan_partials(adg_eval_plan* plan, adg_eval_partials* out);
/* Zero the partials (called by create; call again to re-run). */
adg_status adg_eval_plan_reset(adg_eval_plan* plan);
/* Reset and re-prepare the operands from the same device buffers (their
 * contents may have changed; shapes may not): a repeated evaluation without
 * the plan's allocations and setup.  Device-input plans only. */
adg_status adg_eval_plan_refresh(adg_eval_plan* plan);
/* ADG_ENGINE_SCREEN (default) or ADG_ENGINE_SCREEN_EXACT_HIST for the
 * plan's next runs (set it identically on every rank). */
adg_status adg_eval_plan_set_engine(adg_eval_plan* plan, adg_engine engine);
/* The tile range of `rank` among `world`: contiguous and balanced. */
adg_status adg_eval_plan_shard(adg_eval_plan* plan, int32_t world, int32_t rank, int64_t* tile_begin,
                               int64_t* tile_end);
/* Screen tiles [tile_begin, tile_end) of the plan's tile list. */
adg_status adg_eval_plan_run(adg_eval_plan* plan, int64_t tile_begin, int64_t tile_end);
/* Combine the ranks' partials in place, stream-ordered (no host round
 * trip): [exactly binned edge pairs | histogram] SUM (u64), tile sums SUM
 * (f64: one writer per slot, so exact), [row_max | row_bound] MAX (f32); the
 * exact refine of the row holding the screened maximum, its j chunks split
 * over the ranks and all-gathered; the near-coincident lists all-gathered in
 * fixed 1024-pair blocks and merged in rank order.  A list longer than that
 * is gathered again by the finalize (sized by the largest count), so `comm`
 * must stay valid until adg_eval_plan_finalize returns.  A list over the
 * plan's capacity on any rank makes every rank's finalize redo the histogram
 * in tile chunks, so the report stays bit-identical.  world == 1: no-op. */
adg_status adg_eval_plan_exchange(adg_eval_plan* plan, const adg_collectives* comm);
/* evaluate() over `ndev` GPUs of this process: one rank and one host thread
 * per listed device, each with its own copy of the clouds (host or device
 * pointers; staged per device), NCCL between them (ndev == 1: none).  The
 * GPU-count analogue of the reference's --threads / ADAGIO_THREADS
 * (proj/tools/adagio_main.cpp:501-510, proj/src/parallel.cpp:13-28): the
 * report is bit-identical for any ndev.  All-pairs SCREEN jobs are sharded;
 * EXACT / sampled jobs run on devices[0]. */
adg_status adg_evaluate_multi(int32_t ndev, const int32_t* devices, const void* orig,
                              adg_dtype orig_dtype, int64_t n, int64_t d, const void* emb,
                              adg_dtype emb_dtype, int64_t n_emb, int64_t r,
                              const adg_pair_sampling* mode, int hist_bins, double hist_max,
                              adg_engine engine, adg_report* report, uint64_t* hist_out);
/* Exact refine + deterministic final reduction on the (reduced) partials. */
adg_status adg_eval_plan_finalize(adg_eval_plan* plan, adg_report* report, uint64_t* hist_out);
adg_status adg_eval_plan_destroy(adg_eval_plan* plan);

/* ------------------------------------------------------------ sweeps
 * proj/include/adagio/sweep.hpp + proj/src/sweep.cpp.  The cloud X stays on
 * the device for the whole sweep; every cell's map is applied by the fused
 * transform and scored by the max-only distortion evaluator. */
typedef enum {
  ADG_METHOD_ADAGIO_EXACT = 0,
  ADG_METHOD_ADAGIO_RANDOMIZED = 1,
  ADG_METHOD_PCA = 2,
  ADG_METHOD_JL = 3,
  ADG_METHOD_EXTERNAL = 4
} adg_method;

/* proj/include/adagio/sweep.hpp:19-28 (SweepRow) */
typedef struct {
  int32_t method; /* adg_method */
  int32_t reserved;
  int64_t target_dim;
  uint64_t seed;
  double max_distortion;
  double fit_seconds;
  double eval_seconds;
} adg_sweep_row;

/* proj/include/adagio/sweep.hpp:38-43 (MinDimResult) */
typedef struct {
  int64_t target_dim;
  double achieved_distortion;
  int32_t achieved;
  int32_t monotone;
  int32_t probes;          /* (new) dimensions probed */
  int32_t probes_refined;  /* (new) probes re-evaluated with the exact refine of
                              every candidate row because their bracket
                              [L, U] could not decide a comparison */
} adg_min_dim_result;

/* proj/src/sweep.cpp:142-159: names "adagio_exact", ..., "external";
 * unknown names -> ADG_EINVAL ("unknown method '<name>'"). */
const char* adg_method_name(int32_t method);
adg_status adg_method_from_name(const char* name, int32_t* method_out);

/* proj/src/sweep.cpp:161-201 (tradeoff).  One row per (method, dim, seed) in
 * that nesting order; method external uses the external_rows x external_cols
 * map (fp64, row-major; NULL when absent) once per seed, ignoring dims.
 * rows_out holds rows_capacity rows; *rows_written gets the row count (also
 * when the capacity is too small, then ADG_EINVAL). */
adg_status adg_tradeoff(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                        const int64_t* dims, int64_t n_dims, const int32_t* methods,
                        int64_t n_methods, const uint64_t* seeds, int64_t n_seeds,
                        const adg_pair_sampling* eval_mode, const double* external_map,
                        int64_t external_rows, int64_t external_cols, adg_sweep_row* rows_out,
                        int64_t rows_capacity, int64_t* rows_written);

/* proj/src/sweep.cpp:203-265 (min_dim_for_distortion): exponential probing
 * then bisection on the fixed-seed curve; monotone = no probed value exceeds
 * its smaller-r predecessor by more than 1e-12. */
adg_status adg_min_dim_for_distortion(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n,
                                      int64_t d, int32_t method, double delta, uint64_t seed,
                                      int64_t r_min, int64_t r_max, adg_min_dim_result* out);

/* proj/src/sweep.cpp:267-278 (sweep_csv): bytes needed (excluding NUL). */
size_t adg_sweep_csv(const adg_sweep_row* rows, int64_t count, char* buf, size_t cap);

/* ------------------------------------------- k-NN (downstream.cpp:24-137)
 * Brute force over all database rows with the reference's distance (fp64
 * norm of the row difference) and order ((distance, index), ties toward the
 * smaller index). */

/* proj/src/downstream.cpp:49-60 (knn_query), for nq queries at once:
 * idx_out / dist_out (nq x k, host) receive each query's k nearest rows,
 * ascending. */
adg_status adg_knn_query(adg_ctx* ctx, const void* database, adg_dtype dtype, int64_t n, int64_t d,
                         const void* queries, adg_dtype qdtype, int64_t nq, int64_t qdim, int k,
                         int64_t* idx_out, double* dist_out);

/* proj/src/downstream.cpp:62-88 (majority_classify): labels = database
 * labels (n, NULL -> "database has no labels"); modal label of the pooled
 * neighbour multiset, ties resolved by SeededRng(tie_seed).below. */
adg_status adg_majority_classify(adg_ctx* ctx, const void* queries, adg_dtype qdtype, int64_t nq,
                                 int64_t qdim, const void* database, adg_dtype dtype, int64_t n,
                                 int64_t d, const int32_t* labels, int k, uint64_t tie_seed,
                                 int32_t* label_out);

/* proj/include/adagio/downstream.hpp:14-30 (KnnGraph::Edge, EdgeWeighting) */
typedef struct {
  int32_t u; /* u < v */
  int32_t v;
  double weight;
} adg_knn_edge;
typedef enum { ADG_EDGES_BINARY = 0, ADG_EDGES_GAUSSIAN = 1 } adg_edge_weighting;

/* proj/src/downstream.cpp:90-137 (build_knn_graph): symmetrised union, edges
 * sorted by (u, v); *edges_written = edge count (ADG_EINVAL if it exceeds
 * edges_capacity; n * k always suffices). */
adg_status adg_build_knn_graph(adg_ctx* ctx, const void* X, adg_dtype dtype, int64_t n, int64_t d,
                               int k, int32_t weighting, adg_knn_edge* edges_out,
                               int64_t edges_capacity, int64_t* edges_written);

/* ------------------------------------------------ instrumentation (bench) */
/* Device time (ms) of the last screen-kernel launch on the context stream,
 * measured with CUDA events around that launch only; -1 if none. */
double adg_last_screen_kernel_ms(adg_ctx* ctx);
/* Number of libadg kernels launched by this context since creation. */
uint64_t adg_kernel_launch_count(adg_ctx* ctx);
/* Engine of the last k-NN call on this context: 0 none, 1 fp64 SIMT tiles
 * (knn_query, small graphs), 2 the tensor-core candidate screen (graphs). */
int adg_last_knn_engine(adg_ctx* ctx);
/* MMA passes the last finalized SCREEN evaluation ran over the original
 * coordinates: 1 when every original-side value was exact in the fp16 hi
 * plane (e.g. nearly centred bf16 input, left uncentred), else 3; 0 if none. */
int adg_last_screen_orig_passes(adg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* ADG_H */
