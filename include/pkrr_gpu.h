/*
 * pkrr_gpu.h -- C ABI of the B200 (sm_100a) partitioned Gaussian KRR engine.
 *
 * Drop-in boundary for the reference library's hot path (arxiv 1805.00569
 * reference, /root/reference/proj).  The reference exposes a plain C++ API
 * (no FFI); every entry point below replaces one reference function, cited as
 * file:line, with the same argument meaning and the same error semantics
 * expressed as status codes.  A header-only C++ adapter with the reference's own
 * signatures (pkrr::gpu::gram, cholesky, train_krr, kmeans, make_partition,
 * grid_search, ...) sits on top of this ABI: include/pkrr_gpu.hpp.
 *
 * Conventions
 *  - Matrices are dense row-major FP64 (the reference's Matrix, matrix.hpp:9-28;
 *    its Dataset rows are dense after standardize, dataset.cpp:183-193).
 *  - Every array argument may be a HOST or a DEVICE pointer; the engine detects
 *    which (cudaPointerGetAttributes) and copies only what it must.
 *  - Return value: PKRRGPU_OK (0) or an error status; pkrrgpu_last_error()
 *    returns the message of the last failure on the calling thread.
 *  - Calls on one context are serialised by the caller (like the reference,
 *    which has no globals; runtime.hpp:66-112).
 */
#ifndef PKRR_GPU_H
#define PKRR_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  NPD mirrors NotPositiveDefinite (solver.hpp:17-21); INVALID
 * mirrors std::invalid_argument; LOGIC mirrors kbalance's logic_error
 * (clustering.cpp:172). */
enum pkrrgpu_status {
  PKRRGPU_OK = 0,
  PKRRGPU_INVALID = 1,
  PKRRGPU_NPD = 2,
  PKRRGPU_CUDA = 3,
  PKRRGPU_LOGIC = 4,
  PKRRGPU_IO = 5     /* std::runtime_error of the reference's file IO (open / parse / empty) */
};

/* StrategyKind, same order as strategies.hpp:21. */
enum pkrrgpu_strategy {
  PKRRGPU_EXACT = 0,
  PKRRGPU_DCKRR = 1,
  PKRRGPU_KKRR = 2,
  PKRRGPU_KKRR2 = 3,
  PKRRGPU_KKRR3 = 4,
  PKRRGPU_BKRR = 5,
  PKRRGPU_BKRR2 = 6,
  PKRRGPU_BKRR3 = 7
};

typedef struct pkrrgpu_ctx pkrrgpu_ctx;

/* Engine on one CUDA device (one process per GPU; multi-GPU = one context per
 * rank, see pkrrgpu_grid_args.rank/world). */
int pkrrgpu_create(int device, pkrrgpu_ctx** out);
void pkrrgpu_destroy(pkrrgpu_ctx* ctx);
/* number of visible CUDA devices (0 when there is none) */
int pkrrgpu_device_count(void);
const char* pkrrgpu_last_error(void);
/* Kernel launches made by this context since creation (evidence counter). */
int64_t pkrrgpu_launch_count(const pkrrgpu_ctx* ctx);
const char* pkrrgpu_version(void);

/* ---- kernel (kernel.hpp:40-44) ------------------------------------------ */

/* gram(spec{gaussian, sigma}, A, B) -- kernel.cpp:81-132.  When A == B (same
 * pointer, na == nb) the symmetric path is used: unit diagonal, bitwise
 * symmetric result (kernel.cpp:107-119).  K is na x nb. */
int pkrrgpu_gram(pkrrgpu_ctx* ctx, const double* A, int64_t na, const double* B, int64_t nb,
                 int64_t d, double sigma, double* K);

/* assemble_system(K, lambda, mult) -- kernel.cpp:134-141: A = K + lambda*mult*I. */
int pkrrgpu_assemble(pkrrgpu_ctx* ctx, const double* K, int64_t m, double lambda, int64_t mult,
                     double* A);

/* ---- solver (solver.hpp:29-53) ------------------------------------------- */

/* cholesky(A) -- solver.cpp:13-44.  L lower with zero strict upper triangle.
 * PKRRGPU_NPD: *npd_pivot = first column j whose pivot is !(> 0). */
int pkrrgpu_cholesky(pkrrgpu_ctx* ctx, const double* A, int64_t m, double* L,
                     int64_t* npd_pivot);

/* solve_spd(F, b) -- solver.cpp:46-72: L L^T x = b. */
int pkrrgpu_solve_spd(pkrrgpu_ctx* ctx, const double* L, int64_t m, const double* b, double* x);

/* train_krr(data, spec, lambda) -- solver.cpp:89-125: alpha (m) and the
 * residual ratio ||(K + lambda m I) alpha - y|| / ||y|| (solver.cpp:103-119). */
int pkrrgpu_train_krr(pkrrgpu_ctx* ctx, const double* X, const double* y, int64_t m, int64_t d,
                      double sigma, double lambda, double* alpha, double* residual,
                      int64_t* npd_pivot);

/* KrrModel::predict over q queries -- solver.cpp:74-87:
 * out[j] = sum_i alpha_i k(S_i, Q_j). */
int pkrrgpu_predict(pkrrgpu_ctx* ctx, const double* S, const double* alpha, int64_t m, int64_t d,
                    double sigma, const double* Q, int64_t q, double* out);

/* ---- clustering (clustering.hpp:33-45) ----------------------------------- */

/* kmeans -- clustering.cpp:53-138 (uniform distinct-sample init from
 * Rng(seed), Lloyd, empty-cluster reseed).  Labels are bit-exact with the
 * reference: same distance arithmetic, same tie rule, order-preserving means. */
int pkrrgpu_kmeans(pkrrgpu_ctx* ctx, const double* X, int64_t n, int64_t d, int k, uint64_t seed,
                   double threshold, int max_iters, int32_t* membership, double* centers,
                   int64_t* sizes, int* iterations);

/* kbalance -- clustering.cpp:140-180 (k-means warm start, then the capacity
 * scan replayed exactly in parallel). */
int pkrrgpu_kbalance(pkrrgpu_ctx* ctx, const double* X, int64_t n, int64_t d, int k,
                     uint64_t seed, double threshold, int max_iters, int recompute,
                     int32_t* membership, double* centers, int64_t* sizes);

/* nearest_center for q rows -- clustering.cpp:182-195. */
int pkrrgpu_nearest_center(pkrrgpu_ctx* ctx, const double* centers, int k, int64_t d,
                           const double* Q, int64_t q, int32_t* out);

/* ---- strategies (strategies.hpp:40-120) --------------------------------- */

/* make_partition -- strategies.cpp:64-102 (default KMeansParams, :93-96).
 * part_of[n] = part of each train row; order[n] = rows part by part in
 * within-part order; centers[p*d] for k-means / k-balance (may be NULL);
 * *p_out = effective number of parts (1 for exact). */
int pkrrgpu_make_partition(pkrrgpu_ctx* ctx, int strategy, const double* X, int64_t n, int64_t d,
                           int64_t p, uint64_t seed, int32_t* part_of, int64_t* order,
                           double* centers, int64_t* p_out);

/* Trained per-part models (TrainedPartitions, strategies.hpp:44-47), resident
 * in device memory. */
typedef struct pkrrgpu_models pkrrgpu_models;

/* train_partitions -- strategies.cpp:104-133.  On NPD the status is
 * PKRRGPU_NPD, *failed_part = the first failing part, *npd_pivot its column. */
int pkrrgpu_train_partitions(pkrrgpu_ctx* ctx, int strategy, const double* X, const double* y,
                             int64_t n, int64_t d, int64_t p, uint64_t seed, double sigma,
                             double lambda, pkrrgpu_models** out, int64_t* failed_part,
                             int64_t* npd_pivot);
/* train_partitions(ps, train, spec, lambda, workers) -- strategies.cpp:104-133 with the
 * CALLER's PartitionSet (strategies.hpp:31-36, :50-52): rows = ps.parts concatenated
 * part by part (each part's rows in the caller's order -- make_partition keeps train
 * row order, strategies.cpp:97-99), sizes[p] = the parts' lengths; centers [p*d] or
 * NULL (then predict_nearest raises, like a PartitionSet without centers).  All parts
 * train concurrently on the context's streams, largest first at the highest priority.
 * Errors as pkrrgpu_train_partitions; an empty part or a row outside [0, n) is
 * PKRRGPU_INVALID. */
int pkrrgpu_train_parts(pkrrgpu_ctx* ctx, const double* X, const double* y, int64_t n, int64_t d,
                        const int64_t* rows, const int64_t* sizes, int64_t p, const double* centers, double sigma,
                        double lambda, pkrrgpu_models** out, int64_t* failed_part, int64_t* npd_pivot);
/* Models from host (or device) KrrModels (solver.hpp:37-49): p models of sizes[t] support
 * rows, S = the support rows concatenated model by model (sum(sizes) x d, dense),
 * alpha concatenated the same way, centers [p*d] or NULL, Gaussian sigma. */
int pkrrgpu_models_import(pkrrgpu_ctx* ctx, int64_t p, int64_t d, const int64_t* sizes, const double* S,
                          const double* alpha, const double* centers, double sigma, pkrrgpu_models** out);
/* KrrModel::predict (solver.cpp:74-87) of q rows: model `part` -> out[q]; part = -1:
 * every model, out[t * q + j] (what predict_average / predict_oracle combine,
 * strategies.cpp:135-140 / :151-166). */
int pkrrgpu_models_predict(pkrrgpu_ctx* ctx, const pkrrgpu_models* models, int64_t part, const double* Q,
                           int64_t q, double* out);
/* centers of the partition the models were trained on (p*d), PKRRGPU_INVALID if none */
int pkrrgpu_models_centers(const pkrrgpu_models* models, double* centers);
int64_t pkrrgpu_models_count(const pkrrgpu_models* models);
int64_t pkrrgpu_models_size(const pkrrgpu_models* models, int64_t part);
int pkrrgpu_models_alpha(const pkrrgpu_models* models, int64_t part, double* alpha);
int pkrrgpu_models_residual(const pkrrgpu_models* models, int64_t part, double* residual);
void pkrrgpu_models_free(pkrrgpu_models* models);

/* predict_nearest -- strategies.cpp:142-149 (route by nearest_center, then the
 * chosen model's KrrModel::predict), batched over q queries. */
int pkrrgpu_predict_nearest(pkrrgpu_ctx* ctx, const pkrrgpu_models* models, const double* Q,
                            int64_t q, double* out);

/* grid_search -- strategies.cpp:343-507 (reference signature).  Cells are
 * lambda-major (li * n_sigmas + si, :405).  best_index = first strict minimum
 * over non-failed cells (:499-505), -1 when every cell failed. */
int pkrrgpu_grid_search(pkrrgpu_ctx* ctx, int strategy, const double* X_train,
                        const double* y_train, int64_t n, int64_t d, const double* X_test,
                        const double* y_test, int64_t t, int64_t p, const double* lambdas,
                        int64_t n_lambdas, const double* sigmas, int64_t n_sigmas, uint64_t seed,
                        double* cell_mse, uint8_t* cell_failed, double* cell_residual,
                        int64_t* best_index);

/* All-gather for a sharded partition (one process per GPU): `dev_buf` is a DEVICE
 * buffer of `world` equal slices of `bytes_per_rank` bytes; this rank's slice (offset
 * rank * bytes_per_rank) is filled when the engine calls (its stream synchronised);
 * the callback fills the other slices before returning (e.g. an NCCL all-gather)
 * and returns 0 on success. */
typedef int (*pkrrgpu_allgather_fn)(void* user, void* dev_buf, int64_t bytes_per_rank);

/* Extended grid: adds a held-out evaluation set scored for every cell, explicit
 * k-means parameters, and part sharding for one-process-per-GPU runs. */
typedef struct {
  int strategy;
  const double* X_train;
  const double* y_train;
  int64_t n;
  int64_t d;
  const double* X_test; /* selection set (the reference's "test" argument) */
  const double* y_test;
  int64_t t;
  const double* X_eval; /* optional held-out set; NULL/0 = none */
  const double* y_eval;
  int64_t t_eval;
  int64_t p;
  const double* lambdas;
  int64_t n_lambdas;
  const double* sigmas;
  int64_t n_sigmas;
  uint64_t seed;
  double km_threshold; /* used when km_max_iters > 0; else reference defaults 0.01/100 */
  int km_max_iters;
  int rank;  /* this context trains the parts the LPT rule (m^3, largest first to the least-loaded
              * rank) assigns to `rank` -- identical on every rank (sharding.owned_parts) */
  int world; /* 1 = single process */
  /* optional (world > 1): shard the k-means partition over the ranks -- each rank
   * assigns a 1/world slice of the rows and updates a 1/world slice of the clusters,
   * exchanged by `allgather` every iteration.  Every value is computed by the
   * single-process arithmetic on exactly one rank: bitwise the same partition.
   * NULL: every rank partitions redundantly. */
  pkrrgpu_allgather_fn allgather;
  void* allgather_user;
} pkrrgpu_grid_args;

typedef struct {
  /* per cell [n_lambdas * n_sigmas]; combined over parts only when world == 1 */
  double* cell_mse;
  uint8_t* cell_failed;
  double* cell_residual;
  double* cell_eval_mse; /* optional */
  int64_t best_index;
  /* per (cell, part) [ncell * p], filled for the parts this rank trained; the
   * multi-rank combine sums them in part order (deterministic, GPU-count
   * independent).  All optional. */
  double* part_sse;
  double* part_eval_sse;
  uint8_t* part_failed;
  double* part_residual;
  int64_t* part_test_count;  /* [p] test rows routed to each part */
  int64_t* part_eval_count;  /* [p] */
  /* partition + best-cell predictions, optional */
  int32_t* part_of;      /* [n] */
  double* centers;       /* [p*d] */
  int64_t* part_sizes;   /* [p] */
  double* best_pred;     /* [t] (world == 1) */
  double* best_eval_pred;/* [t_eval] (world == 1) */
  int64_t p_effective;
  /* algorithmic FP64 work done by this rank (SURVEY 8(d) accounting) */
  double flops_chol;
  double flops_gram;
  double flops_other;
  /* optional: this rank's per-cell predictions, [ncell x pred_rows x t] (and t_eval).
   * pred_rows = 1 for the whole / nearest predictors (test-row order; rows routed to
   * parts this rank does not own are 0), = p for average / oracle (one row per part;
   * parts not owned are 0).  Summing them over ranks is exact (disjoint), and
   * pkrrgpu_combine on the sum gives the single-process cell MSEs / best cell bitwise. */
  double* cell_pred;
  double* cell_eval_pred;
  int64_t pred_rows;
} pkrrgpu_grid_out;

int pkrrgpu_grid_search_ex(pkrrgpu_ctx* ctx, const pkrrgpu_grid_args* args,
                           pkrrgpu_grid_out* out);

/* Cell combine + MSE + best cell -- strategies.cpp:458-505 (+ mse :168-177): pred is
 * [ncell x P x t] with P = 1 (whole / nearest: test-row order) or p (average / oracle:
 * one row per part), e.g. the sum over ranks of pkrrgpu_grid_out.cell_pred.  The MSE
 * is summed sequentially in test-row order (the reference's own arithmetic), failed
 * cells (cell_failed may be NULL) get NaN and never win; best = first strict minimum
 * (-1 if none); best_pred (t entries, may be NULL) = the best cell's combined
 * prediction.  grid_search_ex uses the same code for one process. */
int pkrrgpu_combine(pkrrgpu_ctx* ctx, int strategy, int64_t p, int64_t t, int64_t ncell, const double* pred,
                    const double* y, const uint8_t* cell_failed, double* cell_mse, int64_t* best_index,
                    double* best_pred);

/* ---- several GPUs in one process (one host thread per GPU) ----------- */

/* A group of n contexts on devices[0..n) (NULL: 0..n-1), driven by one host thread per
 * GPU.  A device may appear more than once (two contexts sharing one GPU).  Peer
 * access is enabled between distinct devices (NVLink / NVSwitch). */
typedef struct pkrrgpu_multi pkrrgpu_multi;
int pkrrgpu_multi_create(const int* devices, int n, pkrrgpu_multi** out);
void pkrrgpu_multi_destroy(pkrrgpu_multi* m);
int pkrrgpu_multi_size(const pkrrgpu_multi* m);
pkrrgpu_ctx* pkrrgpu_multi_context(pkrrgpu_multi* m, int i);
/* grid_search (strategies.cpp:343-507) over every GPU of the group: each device trains
 * the parts the LPT rule on m^3 gives it (no data-path collective); from 4 devices on
 * (PKRR_SHARD_PARTITION=0/1 forces it) the k-means partition is sharded bit-exactly with a
 * peer-memory all-gather per Lloyd iteration; the devices' per-cell predictions are
 * summed and combined once (pkrrgpu_combine).  args->rank / world / allgather are
 * ignored; `out` is filled as by a one-context call, and is bitwise equal to it. */
int pkrrgpu_multi_grid_search(pkrrgpu_multi* m, const pkrrgpu_grid_args* args, pkrrgpu_grid_out* out);
/* DKRR (the reference's whole-data baseline, runtime.cpp:54-57):
 * train_krr (solver.cpp:89-125) of ONE n-row Gaussian system factorised ACROSS the
 * group's GPUs -- block-cyclic super-columns of 128 G columns stored compactly per GPU
 * (each holds ~1/W of the matrix), each factored panel peer-copied to the other GPUs,
 * lookahead on the next panel's owner, forward substitution fused, backward solve along
 * the owner chain.  alpha (n), residual ||(K + lambda n I) alpha - y|| / ||y||;
 * PKRRGPU_NPD with *npd_pivot = the first failing column.  PKRR_DIST_GROUP sets G. */
int pkrrgpu_multi_train_krr(pkrrgpu_multi* m, const double* X, const double* y, int64_t n, int64_t d,
                            double sigma, double lambda, double* alpha, double* residual, int64_t* npd_pivot);

/* Broadcast of a DEVICE buffer of `bytes` from rank `root` to every rank (e.g. an NCCL
 * broadcast); called with the engine's stream synchronised; returns 0 on success. */
typedef int (*pkrrgpu_bcast_fn)(void* user, void* dev_buf, int64_t bytes, int root);
/* DKRR with one process per GPU: every rank calls it with the same inputs on its own
 * context; rank r stores and updates the super-columns c with c mod world == r, the owner
 * of each step broadcasts its factored panel (with the forward-substitution vector and
 * its NPD status), the backward solve broadcasts each solved block.  alpha (n) and the
 * residual on every rank; NPD as pkrrgpu_train_krr on every rank. */
int pkrrgpu_dist_train_krr(pkrrgpu_ctx* ctx, int rank, int world, pkrrgpu_bcast_fn bcast, void* user,
                           const double* X, const double* y, int64_t n, int64_t d, double sigma, double lambda,
                           double* alpha, double* residual, int64_t* npd_pivot);

/* ---- data preparation (dataset.hpp standardize, strategies.hpp auto_sigma_grid) */

/* standardize -- dataset.cpp:199-232 (+ apply_feature_stats :178-197), dense rows:
 * per-column mean / stddev from the train rows (row-order sums, divisor n, variance
 * clamped at 0), then (x - mean) / stddev for train and test (0 where stddev == 0).
 * Bitwise the reference's.  X_test may be NULL with t = 0; the outputs may alias
 * nothing else; mean_out / stddev_out (d entries) may be NULL. */
int pkrrgpu_standardize(pkrrgpu_ctx* ctx, const double* X_train, int64_t n, int64_t d,
                        const double* X_test, int64_t t, double* train_out, double* test_out,
                        double* mean_out, double* stddev_out);

/* auto_sigma_grid -- strategies.cpp:204-234: min(n, 512) rows drawn by
 * random_permutation(Rng(sub_seed(seed, "sigma-grid"))), the lower median g of their
 * pairwise distances (1 if none or 0), grid_out[e + 4] = g * 2^e for e = -4..4.
 * Bitwise the reference's. */
int pkrrgpu_auto_sigma_grid(pkrrgpu_ctx* ctx, const double* X, int64_t n, int64_t d, uint64_t seed,
                            double* grid_out);

/* load_libsvm -- dataset.cpp:83-125: parse a LIBSVM text file (label, then
 * 1-based strictly increasing index:value pairs; blank lines skipped) with the same
 * strtod/strtol arithmetic and the same errors ("<path>: parse error at line N: ...",
 * "cannot open <path>", "<path>: empty dataset" -> PKRRGPU_IO).  The file is parsed
 * by `threads` host threads (0 = all) into a handle holding the CSR rows exactly as
 * the reference's Dataset stores them; d = 1 + the largest index. */
typedef struct pkrrgpu_dataset pkrrgpu_dataset;
int pkrrgpu_load_libsvm(const char* path, int threads, pkrrgpu_dataset** out);
int pkrrgpu_dataset_shape(const pkrrgpu_dataset* ds, int64_t* n, int64_t* d, int64_t* nnz);
/* the CSR arrays (row_ptr: n + 1 entries, col / val: nnz, y: n), host memory */
int pkrrgpu_dataset_csr(const pkrrgpu_dataset* ds, int64_t* row_ptr, int32_t* col, double* val, double* y);
/* dense row-major n x d rows (absent features 0) and labels, materialised in pinned
 * host staging and copied to X / y (host or device pointers; device: one H2D) */
int pkrrgpu_dataset_dense(pkrrgpu_ctx* ctx, pkrrgpu_dataset* ds, double* X, double* y);
void pkrrgpu_dataset_free(pkrrgpu_dataset* ds);

/* ---- timing hooks (bench / profiling only) ------------------------------- */

/* Device time (ms, CUDA events on the engine's streams) spent in the last
 * grid call by phase: [0] partition, [1] train (gram + Cholesky + solves),
 * [2] solves + predict, [3] total, [4] Cholesky, [5] gram; [8 + t] = when part
 * t's first Cholesky finished, ms after that phase started; [8 + p + 5t .. +4] =
 * part t's first-cell {gram start, gram end, Cholesky start, Cholesky end,
 * predict end}, ms after the call started (n >= 8 + 6p). */
int pkrrgpu_last_timings(const pkrrgpu_ctx* ctx, double* ms, int n);

/* The context's launch stream (cudaStream_t), so callers can time calls with
 * CUDA events on the stream the engine launches on. */
void* pkrrgpu_stream(pkrrgpu_ctx* ctx);

/* Order the context's launch stream after all work already queued on `stream` (a
 * cudaStream_t of the caller, e.g. torch's current stream) -- for device-pointer inputs
 * still being produced there.  Every call reads its inputs on the launch stream. */
int pkrrgpu_wait_stream(pkrrgpu_ctx* ctx, void* stream);

/* FP64 tensor-core peak probe: a DMMA (mma.sync m8n8k4 f64) loop over every
 * SM; *tflops = measured dense FP64 TFLOP/s (roofline denominator). */
int pkrrgpu_fp64_peak(pkrrgpu_ctx* ctx, double* tflops);

/* Roofline probe of the dominant kernel: factor an m x m SPD system alone on one
 * stream with CUDA events around every trailing-SYRK launch.  out[0] total ms,
 * out[1] Cholesky algorithmic flops, out[2] SYRK ms (sum over launches),
 * out[3] SYRK algorithmic flops, out[4] SYRK launches, out[5] NPD flag.
 * alone != 0: the panel schedule of a system factorised alone (single-part grids,
 * pkrrgpu_cholesky, pkrrgpu_train_krr), else the one of a part among several. */
int pkrrgpu_probe_potrf(pkrrgpu_ctx* ctx, int64_t m, int alone, double* out);

#ifdef __cplusplus
}
#endif
#endif /* PKRR_GPU_H */
