// kernels.cuh -- launch wrappers for the sm_100a kernels of the pkrr engine.
// All launchers are asynchronous on the given stream and count launches in
// *launches (evidence for bench.py's gpu_launches).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>
#include <vector>

namespace pk {

constexpr int kNB = 128;  // Cholesky block (leaf / panel) size; parts are padded to it

// Launch evidence + launch-error capture.  Every launcher calls launched() right after
// its kernel launch(es): the count feeds bench.py's gpu_launches, and the first
// launch error since reset() (cudaGetLastError: bad configuration, missing smem
// attribute, ...) is kept so the C ABI returns PKRRGPU_CUDA instead of OK with
// garbage outputs.  fault_at (PKRR_FAULT_LAUNCH, test hook) turns the launch with
// that running count into an invalid one.
struct Counter {
  int64_t launches = 0;
  cudaError_t err = cudaSuccess;
  int64_t err_at = 0;    // launch count at which err was seen
  int64_t fault_at = 0;
  void launched(int k = 1);
  void reset();
};

// ---- TMA descriptors -------------------------------------------------------
bool make_tmap(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld);

// ---- row norms: out[i] = sum_k x_ik^2, sequential, no FMA (dataset.cpp:49-53)
void launch_row_norms(const double* X, int64_t rows, int64_t d, int64_t ld, double* out,
                      cudaStream_t s, Counter& c);

// ---- gather rows idx[0..cnt) of X (n x d) into dst (rows_pad x dp), zero padded
void launch_gather_rows(const double* X, int64_t d, const int64_t* idx, int64_t cnt,
                        double* dst, int64_t rows_pad, int64_t dp, cudaStream_t s, Counter& c);
void launch_gather_vec(const double* y, const int64_t* idx, int64_t cnt, double* dst,
                       int64_t pad, cudaStream_t s, Counter& c);

// ---- DMMA GEMM family (gemm_dmma.cuh) -------------------------------------
// K (ldk x ldk, padded mp) = gaussian gram of Xp (mp x dp) ; valid = m
// With A != null the lower tiles of A = K + shift I (strategies.cpp:296-303, the first lambda's
// system) are written by the same epilogue when the ping-pong kernel runs; returns whether A
// was written (otherwise launch_assemble forms it).
bool launch_gram_sym(const CUtensorMap& tmX, const double* norms, int64_t mp, int64_t dp,
                     int64_t m, double sigma, double* K, int64_t ldk, const int* abort,
                     cudaStream_t s, Counter& c, bool mirror = true, double* A = nullptr, double shift = 0.0);
// Kc (qp x mp) = k(Q_q, X_i); valid rows q, valid cols m
void launch_gram_cross(const CUtensorMap& tmQ, const CUtensorMap& tmX, const double* qnorms,
                       const double* xnorms, int64_t qp, int64_t q, int64_t mp, int64_t m,
                       int64_t dp, double sigma, double* Kc, cudaStream_t s, Counter& c);
// Blocked right-looking Cholesky of A (mp x mp, lower, mp % 128 == 0) in place.
// Linv: mp x 128 scratch receiving inv(L_kk) per diagonal block.
// status[0] = abort flag, status[1] = first failing global column (int).
// slices/exps: int8 [8 x mp x 512] and int [mp] scratch for the Ozaki SYRK mode (may be null).
void shadow_report();  // PKRR_SHADOW debug mode (see launch_potrf)
// Forward substitution fused into the factorization: w (mp) := y, then each panel's
// leaf sets z_k = inv(L_kk) w_k and its TRSM subtracts L21 z_k from w below it, so
// z = L^{-1} y is complete with the factor (launch_trsv_bwd finishes the solve).
struct FwdSolve {
  const double* y;
  double* w;
  double* z;
};
// Kernel-matrix build fused into the factorization (the dataflow path only): A and K
// are formed tile by tile from the padded rows (tmX over Xp [mp x dp], norms) as
// K = exp(-d^2 / ((2 sigma) sigma)), A = K + shift I, instead of gram + assemble kernels.
struct GramFuse {
  CUtensorMap tmX;
  const double* xnorm;
  double* K;
  int64_t dp;
  int64_t m_valid;
  double sigma;
  double shift;
};
// true when launch_potrf factors an mp x mp system with the dataflow kernel
// (csrc/potrf_df.cuh): a system factorised alone (latency) with mp < 8192, default
// schedule settings (PKRR_DF=0 disables it)
bool potrf_df_eligible(int64_t mp, bool latency);
// Returns true when the forward solve was fused (fs given and not in PKRR_SHADOW mode).
// gf (eligible systems only, else ignored): A is built from gf instead of read.
bool launch_potrf(double* A, const CUtensorMap& tmA, const CUtensorMap& tmLinv, double* Linv,
                  int64_t mp, int64_t m_valid, int* status, cudaStream_t s, Counter& c,
                  int8_t* slices = nullptr, int* exps = nullptr, cudaStream_t s2 = nullptr,
                  bool latency = false, const FwdSolve* fs = nullptr, const GramFuse* gf = nullptr);
// s2 (optional): a second stream for lookahead -- the next panel's columns are
// updated first on s and the rest of the trailing update runs on s2, overlapping the
// next panel factorisation; the result is bitwise the same as without.
// latency: the system is factorised alone (nothing else to fill the GPU): small
// systems (m < 8192) then use single-panel groups (see launch_potrf).
// Number of 128-column panels per trailing update (K = 128 * G); 0 (default) = automatic:
// 4 for m < 8192 or the int8 update, 8 below m = 16384, 16 above (max 16).
void set_panel_group(int g);
// SYRK grid: 0 = one 128x128 tile per CTA (default), 1 = persistent (one CTA per SM).
void set_syrk_persistent(int on);
// Trailing SYRK on the int8 tensor cores (tcgen05 kind::i8, Ozaki splitting into 8
// 7-bit slices, FP64-accurate) when 1; DMMA f64 when 0 (default).
void set_syrk_ozaki(int on);
int syrk_ozaki();
// Probe hook: when set, every trailing-SYRK launch is bracketed by events and its
// algorithmic flop count recorded (used by pkrrgpu_probe_potrf only).
void set_syrk_probe(std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* ev, std::vector<double>* flops);
// Recompute inv(L_kk) for every diagonal block of an existing factor.
void launch_diag_inverses(const double* L, int64_t mp, double* Linv, cudaStream_t s, Counter& c);
// Zero the strict upper triangle (API parity with solver.cpp:34).
void launch_zero_upper(double* A, int64_t mp, cudaStream_t s, Counter& c);

// ---- triangular solves (L L^T x = b) on the blocked factor ----------------
// scratch: 2*nb + 2 ints (tickets + flags), zeroed by the launcher
size_t trsv_scratch_ints(int64_t mp);  // ints of the solves' scratch (tickets, flags, tagged x words)
void launch_trsv(const double* L, const double* Linv, int64_t mp, const double* b, double* z,
                 double* x, int* scratch, const int* abort, cudaStream_t s, Counter& c);
// backward half only (z from a fused forward substitution)
void launch_trsv_bwd(const double* L, const double* Linv, int64_t mp, const double* z, double* x,
                     int* scratch, const int* abort, cudaStream_t s, Counter& c);

// ---- assemble: A = K + shift * I (full copy) ------------------------------
// y = K alpha from the lower 128x128 tiles of a symmetric K (mp x mp, ld = mp); deterministic.
// y holds kSymvSplit partial vectors of mp (tile ranges split over that many CTAs per
// block row, so the latency-bound GEMV occupies its SMs a quarter as long);
// launch_residual_finish sums them in a fixed order.
constexpr int kSymvSplit = 4;
void launch_symv_lower(const double* K, int64_t mp, const double* alpha, double* y, const int* abort,
                       cudaStream_t s, Counter& c);
void launch_assemble(const double* K, double* A, int64_t mp, double shift, const int* abort,
                     cudaStream_t s, Counter& c, bool lower_only = false);

// ---- GEMV rows: out[i] = sum_{j<cols} M[i][j] v[j], i < rows (deterministic)
// prediction with the cross kernel tile fused into the alpha contraction
// (predict_fused.cuh); partial = predict_partial_elems(qp, mp) doubles of scratch
int64_t predict_partial_elems(int64_t qp, int64_t mp);
void launch_predict_fused(const CUtensorMap& tmQ, const CUtensorMap& tmX, const double* qnorms,
                          const double* xnorms, int64_t qp, int64_t q, int64_t mp, int64_t m, int64_t dp,
                          double sigma, const double* alpha, double* partial, double* pred, const int* abort,
                          cudaStream_t s, Counter& c);
void launch_gemv_rows(const double* M, int64_t ld, int64_t rows, int64_t cols, const double* v,
                      double* out, const int* abort, cudaStream_t s, Counter& c);
// residual ratio of (K + shift I) alpha = y from Kalpha (strategies.cpp:310-320 and
// solver.cpp:103-119): out[0] = sqrt(res/yy), out[1] = sqrt(res)/sqrt(yy)
void launch_residual_finish(const double* Kalpha, const double* alpha, const double* y,
                            int64_t m, double shift, double* out, const int* abort,
                            cudaStream_t s, Counter& c);
// pred rows -> scatter to test order (pred_all[pos[j]] = pred[j]) and
// sse = sum (pred_j - ytest[pos[j]])^2 (fixed-order tree), out[0] = sse
void launch_sse_scatter(const double* pred, const int64_t* pos, int64_t cnt, const double* ytest,
                        double* pred_all, double* out, const int* abort, cudaStream_t s,
                        Counter& c);
// combine per-part predictions (average / oracle / nearest / whole) in part order
// into pred[t] and mse over all rows (strategies.cpp:458-495)
// every cell's combined prediction and its reference-order MSE (strategies.cpp:458-495,
// mse :168-177): pp [ncell x P x t]; predictor 0 whole, 1 average (x 1/p), 2 nearest,
// 3 oracle, 4 average by division (predict_average); comb [ncell x t], mse [ncell]
void launch_combine_cells(const double* pp, int64_t P, int64_t t, int64_t ncell, int predictor, const double* y,
                          double* comb, double* mse, cudaStream_t s, Counter& c);
void launch_combine(const double* pp, int64_t p, int64_t t, int predictor, const int32_t* route,
                    const double* ytest, double* pred, double* mse_out, cudaStream_t s,
                    Counter& c);

// ---- clustering (bit-exact with clustering.cpp) ---------------------------
// mode 0: kmeans assign (all clusters, min_j init 0, counts changes)
// mode 1: kbalance re-argmin over open clusters for rows in [row0, n) whose
//         current choice is closed (or < 0), min_j init -1
void launch_assign(const double* X, int64_t n, int64_t d, const double* xnorm,
                   const double* centers, const double* cnorm, int k, int mode,
                   const uint8_t* open, int64_t row0, int32_t* label, double* best_dist,
                   unsigned long long* changed, cudaStream_t s, Counter& c);
// stable grouping of rows by label: sizes[k], start[k], members[n] (row order)
// tmp: >= (ceil(n/256) * k + 2k) int64
void launch_group(const int32_t* label, int64_t n, int k, int64_t* sizes, int64_t* start,
                  int64_t* members, int64_t* tmp, cudaStream_t s, Counter& c);
// centers[j][f] = (sum over members in row order) * (1.0 / size)  (clustering.cpp:34-49)
// (clusters [j0, j1) only when given: one rank's share of a sharded update)
void launch_means(const double* X, int64_t d, const int64_t* members, const int64_t* start,
                  const int64_t* sizes, int k, double* centers, cudaStream_t s, Counter& c, int j0 = 0,
                  int j1 = -1);
// count of i < n with a[i] != b[i] (the k-means "changed" count of a sharded assign)
void launch_label_diff(const int32_t* a, const int32_t* b, int64_t n, unsigned long long* count,
                       cudaStream_t s, Counter& c);
// argmax_i best[i] over rows whose cluster has size > 1 (first index on ties)
void launch_farthest(const double* best, const int32_t* label, const int64_t* sizes, int64_t n,
                     unsigned long long* out, cudaStream_t s, Counter& c);
// histogram of label[row0..row1] (inclusive) into hist[k] (zeroed by launcher)
void launch_hist(const int32_t* label, int64_t row0, int64_t row1, int k, int64_t* hist,
                 cudaStream_t s, Counter& c);
// per-cluster position of the thr[j]-th occurrence of j in label[row0..n)
void launch_events(const int32_t* label, int64_t row0, int64_t n, int k, const int64_t* thr,
                   int64_t* pos, cudaStream_t s, Counter& c);

// FP64 DMMA throughput probe (8 independent accumulator chains per warp)
void launch_dmma_probe(int blocks, int threads, int iters, double* sink, cudaStream_t s, Counter& c);

// ---- data preparation ----
// column mean / stddev of X (n x d, row pitch ld), bit-exact with dataset.cpp:199-224;
// false if X / ld do not meet TMA alignment (16-byte base, even ld)
bool launch_standardize_stats(const double* X, int64_t n, int64_t d, int64_t ld, double* mean, double* stddev,
                              cudaStream_t s, Counter& c);
// out = (X - mean) / stddev per column, 0 where stddev == 0 (dataset.cpp:187-194)
void launch_standardize_apply(const double* X, int64_t n, int64_t d, const double* mean, const double* stddev,
                              double* out, cudaStream_t s, Counter& c);
// auto_sigma_grid's pairwise distances in the reference's push order (strategies.cpp:214-222)
void launch_pair_dist(const double* G, const double* norms, int64_t cnt, int64_t d, double* out, cudaStream_t s,
                      Counter& c);

// ---- distributed factorization building blocks (csrc/dist.cu) ----------------
// C[c_row0 + .., c_col0 + ..] -= A[a_row0 + .., a_k0 ..] B[b_row0 + .., b_k0 ..]^T over
// tiles_m128 x tiles_n tiles of 128 x 128, K = 16 ktiles
void launch_gemm_update(const CUtensorMap& tmA, const CUtensorMap& tmB, int a_row0, int a_k0, int b_row0, int b_k0,
                        int ktiles, double* C, int64_t ldc, int c_row0, int c_col0, int tiles_m128, int tiles_n,
                        const int* abort, cudaStream_t s, Counter& c);
// panel TRSM in place: C[row0 .., col0 .. +128] = A[row0 .., col0 ..] inv(L_kb)^T over
// rows128 128-row blocks; fused forward substitution fw -= C fz (fz = z + 128 kb)
void launch_gemm_trsm(const CUtensorMap& tmA, const CUtensorMap& tmLinv, int row0, int col0, int kb, int rows128,
                      double* C, int64_t ldc, const double* fz, double* fw, const int* abort, cudaStream_t s,
                      Counter& c);
// the Cholesky leaf of global block kb of a matrix whose block (kb, kb) sits at
// A_shifted + 128 kb (lda + 1)
void launch_leaf_at(double* A_shifted, int64_t lda, int kb, double* Linv, int* status, int64_t m_valid,
                    const double* w, double* z, cudaStream_t s, Counter& c);
void launch_gram_block(const CUtensorMap& tmX, const double* norms, int64_t dp, int row0, int col0, int rows,
                       int cols, int64_t m_valid, double sigma, double* Cblk, int64_t ldc, cudaStream_t s,
                       Counter& c);
void launch_set_diag(double* A, int64_t ld, int64_t row0, int64_t col0, int64_t count, double v, cudaStream_t s,
                     Counter& c);
// backward solve of blocks [ilo, ihi) (x blocks >= ihi final); scratch: nb + 1 ints
void launch_trsv_bwd_range(const double* L_shifted, int64_t ld, const double* Linv, const double* z, double* x, int nb,
                           int ilo, int ihi, int* scratch, const int* abort, cudaStream_t s, Counter& c);
}  // namespace pk
