// kernels.cu -- sm_100a kernels of the pkrr engine (everything except the DMMA
// GEMM template, which lives in gemm_dmma.cuh and is instantiated here).
//
// Bit-exactness: the clustering kernels (norms, assign, means) use explicit
// __dmul_rn/__dadd_rn so nvcc cannot contract to FMA; together with the
// reference's summation order this makes partition labels bit-identical to
// clustering.cpp.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cstdlib>
#include <atomic>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>

#include "gemm_dmma.cuh"
#include "syrk_persistent.cuh"
#include "ozaki_syrk.cuh"
#include "predict_fused.cuh"
#include "gram_pp.cuh"
#include <string>
#include "kernels.cuh"

namespace pk {

// ---------------------------------------------------------------------------
// per-device state.  Several contexts (one host thread per GPU, pkrrgpu_multi) can
// launch concurrently on different devices: the SM count and the >48 KB dynamic
// shared-memory opt-ins are per device, never per process.
// ---------------------------------------------------------------------------
static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & 63;
}

int sm_count() {
  static std::atomic<int> sms[64];
  const int dev = current_device();
  int v = sms[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}
#define g_sms (::pk::sm_count())

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device).  The bit
// is set after the call, so a concurrent first launch on the same device sets it too.
template <typename F>
static void smem_optin(std::atomic<uint64_t>& done, F* kernel, int bytes) {
  const uint64_t bit = 1ull << current_device();
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.fetch_or(bit, std::memory_order_acq_rel);
}

__global__ void fault_probe_kernel() {}

void Counter::launched(int k) {
  const int64_t before = launches;
  launches += k;
  if (fault_at > 0 && before < fault_at && launches >= fault_at)
    fault_probe_kernel<<<1, 4096>>>();  // 4096 threads per block: cudaErrorInvalidConfiguration
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err == cudaSuccess) {
    err = e;
    err_at = launches;
  }
}

void Counter::reset() {
  cudaGetLastError();  // a stale error of an earlier call is not this call's
  err = cudaSuccess;
  err_at = 0;
}

// ---------------------------------------------------------------------------
// TMA descriptors (driver entry point fetched through the runtime)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool make_tmap(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 8)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), 64u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// ---------------------------------------------------------------------------
// row norms (dataset.cpp:49-53 squared_norm; clustering.cpp:28-32)
// ---------------------------------------------------------------------------
constexpr int kNormRows = 128, kChunk = 32;

__global__ void __launch_bounds__(kNormRows) row_norms_kernel(const double* __restrict__ X,
                                                               int64_t rows, int64_t d, int64_t ld,
                                                               double* __restrict__ out) {
  __shared__ double xs[kNormRows][kChunk + 1];
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kNormRows;
  const int64_t i = r0 + threadIdx.x;
  double s = 0.0;
  for (int64_t c0 = 0; c0 < d; c0 += kChunk) {
    const int cw = static_cast<int>(d - c0 < kChunk ? d - c0 : kChunk);
    __syncthreads();
    {
      double v[kChunk];
      const int cc = threadIdx.x & (kChunk - 1), rb = threadIdx.x / kChunk;
#pragma unroll
      for (int u = 0; u < kChunk; ++u) {
        const int64_t gr = r0 + rb + u * (kNormRows / kChunk);
        v[u] = (gr < rows && cc < cw) ? __ldg(X + gr * ld + c0 + cc) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kChunk; ++u) xs[rb + u * (kNormRows / kChunk)][cc] = v[u];
    }
    __syncthreads();
    for (int cc = 0; cc < cw; ++cc) {
      const double v = xs[threadIdx.x][cc];
      s = __dadd_rn(s, __dmul_rn(v, v));
    }
  }
  if (i < rows) out[i] = s;
}

void launch_row_norms(const double* X, int64_t rows, int64_t d, int64_t ld, double* out,
                      cudaStream_t s, Counter& c) {
  if (rows <= 0) return;
  row_norms_kernel<<<static_cast<unsigned>((rows + kNormRows - 1) / kNormRows), kNormRows, 0, s>>>(
      X, rows, d, ld, out);
  c.launched();
}

// ---------------------------------------------------------------------------
// gathers
// ---------------------------------------------------------------------------
__global__ void gather_rows_kernel(const double* __restrict__ X, int64_t d,
                                   const int64_t* __restrict__ idx, int64_t cnt,
                                   double* __restrict__ dst, int64_t rows_pad, int64_t dp) {
  const int64_t total = rows_pad * dp;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / dp, col = e % dp;
    dst[e] = (r < cnt && col < d) ? X[idx[r] * d + col] : 0.0;
  }
}

void launch_gather_rows(const double* X, int64_t d, const int64_t* idx, int64_t cnt, double* dst,
                        int64_t rows_pad, int64_t dp, cudaStream_t s, Counter& c) {
  const int64_t total = rows_pad * dp;
  if (total <= 0) return;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  gather_rows_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(X, d, idx, cnt, dst, rows_pad, dp);
  c.launched();
}

__global__ void gather_vec_kernel(const double* __restrict__ y, const int64_t* __restrict__ idx,
                                  int64_t cnt, double* __restrict__ dst, int64_t pad) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < pad) dst[i] = i < cnt ? y[idx[i]] : 0.0;
}

void launch_gather_vec(const double* y, const int64_t* idx, int64_t cnt, double* dst, int64_t pad,
                       cudaStream_t s, Counter& c) {
  if (pad <= 0) return;
  gather_vec_kernel<<<static_cast<unsigned>((pad + 255) / 256), 256, 0, s>>>(y, idx, cnt, dst, pad);
  c.launched();
}

// ---------------------------------------------------------------------------
// DMMA GEMM launches
// ---------------------------------------------------------------------------
// Launch with programmatic stream serialization: the kernel's CTAs may be scheduled
// while the previous kernel in the stream drains (every kernel of the factorisation
// chain starts with pdl_wait), trimming the launch gap between dependent panel steps.
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static const bool off = std::getenv("PKRR_PDL") && std::atoi(std::getenv("PKRR_PDL")) == 0;
  cfg.numAttrs = off ? 0 : 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int BM, int MODE>
static void gemm_launch(const CUtensorMap& a, const CUtensorMap& b, const GemmParams& p,
                        int blocks, cudaStream_t s, Counter& c) {
  if (blocks <= 0) return;
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, dgemm_tn_kernel<BM, MODE>, GemmCfg<BM>::SMEM);
  launch_pdl(dgemm_tn_kernel<BM, MODE>, blocks, gemm_threads<MODE>(), GemmCfg<BM>::SMEM, s, a, b, p);
  c.launched();
}

bool launch_gram_sym(const CUtensorMap& tmX, const double* norms, int64_t mp, int64_t dp,
                     int64_t m, double sigma, double* K, int64_t ldk, const int* abort,
                     cudaStream_t s, Counter& c, bool mirror, double* A, double shift) {
  GemmParams p{};
  p.mirror = mirror ? 1 : 0;
  p.a_row0 = p.b_row0 = 0;
  p.a_k0 = p.b_k0 = 0;
  p.ktiles = static_cast<int>(dp / kBK);
  p.C = K;
  p.ldc = ldk;
  const int T = static_cast<int>(mp / 128);
  p.tiles_m = p.tiles_n = T;
  p.lower = 1;
  p.norm_a = p.norm_b = norms;
  p.valid_a = p.valid_b = static_cast<int>(m);
  p.denom = (2.0 * sigma) * sigma;
  p.neg_inv_denom = -1.0 / p.denom;
  p.abort_flag = abort;
  static const bool pp = !(std::getenv("PKRR_GRAM_PP") && std::atoi(std::getenv("PKRR_GRAM_PP")) == 0);
  if (!mirror && pp) {
    // the pipeline's K (lower tiles only): persistent ping-pong kernel (gram_pp.cuh)
    GramPPParams q{};
    q.T = T;
    q.ktiles = p.ktiles;
    q.K = K;
    q.ldk = ldk;
    q.norms = norms;
    q.valid = static_cast<int>(m);
    q.neg_inv_denom = p.neg_inv_denom;
    q.abort_flag = abort;
    q.A = A;
    q.shift = shift;
    // alternate the warpgroups' mainloops strictly while the epilogue is comparable to the
    // mainloop (dp <= 256); with long mainloops (C4: dp = 784) two concurrent mainloops hide
    // each other's latencies better than one at a time
    static const int turn_max = std::getenv("PKRR_GRAM_TURNS") ? std::atoi(std::getenv("PKRR_GRAM_TURNS")) : 16;
    q.turns = q.ktiles <= turn_max ? 1 : 0;
    static std::atomic<uint64_t> attr{0};
    smem_optin(attr, gram_pp_kernel, kPPSmem);
    const int nhalf = T * (T + 1);
    launch_pdl(gram_pp_kernel, static_cast<unsigned>(nhalf < g_sms ? nhalf : g_sms), kPPThreads, kPPSmem, s, tmX, q);
    c.launched();
    return A != nullptr;
  }
  gemm_launch<128, G_GRAM_SYM>(tmX, tmX, p, T * (T + 1) / 2, s, c);
  return false;
}

void launch_gram_cross(const CUtensorMap& tmQ, const CUtensorMap& tmX, const double* qnorms,
                       const double* xnorms, int64_t qp, int64_t q, int64_t mp, int64_t m,
                       int64_t dp, double sigma, double* Kc, cudaStream_t s, Counter& c) {
  GemmParams p{};
  p.ktiles = static_cast<int>(dp / kBK);
  p.C = Kc;
  p.ldc = mp;
  p.tiles_m = static_cast<int>(qp / 64);
  p.tiles_n = static_cast<int>(mp / 128);
  p.norm_a = qnorms;
  p.norm_b = xnorms;
  p.valid_a = static_cast<int>(q);
  p.valid_b = static_cast<int>(m);
  p.denom = (2.0 * sigma) * sigma;
  p.neg_inv_denom = -1.0 / p.denom;
  gemm_launch<64, G_GRAM_CROSS>(tmQ, tmX, p, p.tiles_m * p.tiles_n, s, c);
}

int64_t predict_partial_elems(int64_t qp, int64_t mp) { return qp * (mp / 128); }

void launch_predict_fused(const CUtensorMap& tmQ, const CUtensorMap& tmX, const double* qnorms,
                          const double* xnorms, int64_t qp, int64_t q, int64_t mp, int64_t m, int64_t dp,
                          double sigma, const double* alpha, double* partial, double* pred, const int* abort,
                          cudaStream_t s, Counter& c) {
  if (q <= 0) return;
  PredictParams p{};
  p.ktiles = static_cast<int>(dp / kBK);
  p.tiles_q = static_cast<int>(qp / 64);
  p.tiles_x = static_cast<int>(mp / 128);
  // about two CTAs per SM over the whole launch, at least one support tile each
  int nch = (2 * g_sms + p.tiles_q - 1) / p.tiles_q;
  nch = nch < 1 ? 1 : (nch > p.tiles_x ? p.tiles_x : nch);
  p.chunk = (p.tiles_x + nch - 1) / nch;
  nch = (p.tiles_x + p.chunk - 1) / p.chunk;
  p.valid_x = static_cast<int>(m);
  p.qp = qp;
  p.qnorms = qnorms;
  p.xnorms = xnorms;
  p.alpha = alpha;
  p.neg_inv_denom = -1.0 / ((2.0 * sigma) * sigma);
  p.partial = partial;
  p.abort_flag = abort;
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, predict_fused_kernel, GemmCfg<64>::SMEM);
  predict_fused_kernel<<<p.tiles_q * nch, kGemmThreads, GemmCfg<64>::SMEM, s>>>(tmQ, tmX, p);
  predict_reduce_kernel<<<static_cast<unsigned>((q + 255) / 256), 256, 0, s>>>(partial, qp, nch, q, pred, abort);
  c.launched(2);
}

// ---------------------------------------------------------------------------
// Cholesky leaf (128 x 128 diagonal block), one CTA of 8 warps:
//   for each 32-column panel: warp 0 factors the 32x32 diagonal block in registers
//   while warps 1..3-pb factor the rows below it column by column from the values
//   warp 0 publishes (so no panel TRSM, and no 32x32 inverse, on the chain), then a
//   register-blocked DMMA SYRK inside smem; warp 7 inverts each 32x32 diagonal block
//   off the chain; finally the blocked inverse of the whole 128 block (DMMA) for the
//   panel TRSM of the outer algorithm and for the triangular solves.
// Pivot test / sqrt / column divide / rank-1 update per column follow
// solver.cpp:18-33; only the blocking (summation order) differs.
// ---------------------------------------------------------------------------
constexpr int kLeafThreads = 256;
constexpr int kLS = 132;  // S stride (doubles): == 4 (mod 16) -> conflict-free DMMA fragments
constexpr int kBS = 36;   // 32x32 block stride
constexpr int kLeafSmem = (kNB * kLS + 4 * 32 * kBS + 3 * 32 * kBS) * 8 + (1 + 32 + 4) * 8 + 16;

// Register-blocked variants (one A fragment feeds several DMMAs: half the LDS traffic,
// which otherwise co-limits with the single SM's DMMA rate):
// acc[c] (8x8) += A(rows, k) * Bt(rows 8c.., k)^T, c < 4 (one row tile x 4 column tiles)
__device__ __forceinline__ void mma_row4_rt(double (&acc)[4][2], const double* A, int lda, const double* Bt,
                                            int ldb, int k0, int k1, int lr, int lk) {
#pragma unroll 4
  for (int k = k0; k < k1; k += 4) {
    const double a = A[lr * lda + k + lk];
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma(acc[c], a, Bt[(8 * c + lr) * ldb + k + lk]);
  }
}
// acc[r][c] (2x2 tiles of 8x8) += A(rows 8r.., k) * Bt(rows 8c.., k)^T
__device__ __forceinline__ void mma_2x2_rt(double (&acc)[2][2][2], const double* A, const double* Bt, int ld,
                                           int K, int lr, int lk) {
#pragma unroll 4
  for (int k = 0; k < K; k += 4) {
    const double a0 = A[lr * ld + k + lk], a1 = A[(8 + lr) * ld + k + lk];
    const double b0 = Bt[lr * ld + k + lk], b1 = Bt[(8 + lr) * ld + k + lk];
    dmma(acc[0][0], a0, b0);
    dmma(acc[0][1], a0, b1);
    dmma(acc[1][0], a1, b0);
    dmma(acc[1][1], a1, b1);
  }
}
// acc[c] (8x8) += A(rows, k) * B(k, cols 8c..) with B row-major [k][n], k in [k0, k1)
__device__ __forceinline__ void mma_row4_rn(double (&acc)[4][2], const double* A, int lda, const double* B,
                                            int ldb, int k0, int k1, int lr, int lk) {
#pragma unroll 4
  for (int k = k0; k < k1; k += 4) {
    const double a = A[lr * lda + k + lk];
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma(acc[c], a, B[(k + lk) * ldb + 8 * c + lr]);
  }
}

// the same with a lower-triangular B (B[k][n] = 0 for n > k, a D block): column tile c
// only meets k >= 8 c, so those DMMAs are not issued (K = 32)
__device__ __forceinline__ void mma_row4_rn_lowB(double (&acc)[4][2], const double* A, int lda, const double* B,
                                                 int ldb, int lr, int lk) {
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    const double a = A[lr * lda + k + lk];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (k + 4 > 8 * c) dmma(acc[c], a, B[(k + lk) * ldb + 8 * c + lr]);
  }
}

// lane i owns row i of the 32x32 block at Sd (stride kLS); returns the first
// failing column or -1 (solver.cpp:18-33 per column: test, sqrt, divide, update).
// Column values are broadcast through shared memory, one 40-double slot per column
// (`col`, 16-byte aligned; slot j+1 holds column j's l values and pivot j+1): one STS
// per lane, then LDS.128 reads of two values each, instead of two SHFL.IDX per double.
// Lane j+1 updates its own next pivot at once (its a[j+1] -= l*l is exactly the
// general update with l_k = its own l) and publishes it with the column, so the pivot
// chain is LDS -> rsqrt -> multiply -> STS -> syncwarp.  After each column lane 0
// arrives on cbar[j] (when given): the warps factoring the rows below the block
// (warp_tall32) read the same slots without ever holding this warp up.
template <int LS>
__device__ __noinline__ int warp_potrf32_s(double* Sd, double* col, uint64_t* cbar, int lane) {
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = Sd[lane * LS + c];
  int bad = -1;
  if (lane == 0) col[32] = a[0];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const double* cur = col + j * 40;
    double* nxt = col + (j + 1) * 40;
    double piv = cur[32];
    if (!(piv > 0.0) && bad < 0) bad = j;
    piv = bad >= 0 ? 1.0 : piv;  // keep the warp going; the result is discarded
    // one reciprocal square root on the pivot chain instead of sqrt + divide
    const double rj = rsqrt(piv);
    const double dj = piv * rj;
    const double l = a[j] * rj;
    a[j] = lane == j ? dj : (lane > j ? l : 0.0);
    if (lane == j + 1) {
      a[j + 1] = a[j + 1] - l * l;
      nxt[32] = a[j + 1];
    }
    nxt[lane] = l;
    __syncwarp();
    if (cbar && lane == 0) mbar_arrive_nomem(&cbar[j]);
    if (j + 1 < 32) {
      // rows k > j: a[k] -= l_i * l_k (lane j+1's own diagonal already done).  Applied
      // to every lane: entries above a lane's diagonal (k > i) only collect values that
      // are never read (a later column zeroes them, the final store drops them), and
      // the valid entries combine valid values only -- no per-entry selects, about a
      // third of the code (the leaf is instruction-fetch bound when its SM is cold).
#pragma unroll
      for (int k = (j + 1) & ~1; k < 32; k += 2) {
        const double2 lk = *reinterpret_cast<const double2*>(nxt + k);
        if (k > j) a[k] = (k == j + 1 && lane == j + 1) ? a[k] : a[k] - l * lk.x;
        if (k + 1 > j) a[k + 1] -= l * lk.y;
      }
    }
  }
  if (bad < 0) {
#pragma unroll
    for (int c = 0; c < 32; ++c) Sd[lane * LS + c] = c <= lane ? a[c] : 0.0;
  }
  return bad;
}
__device__ __forceinline__ int warp_potrf32(double* Sd, double* col, uint64_t* cbar, int lane) {
  return warp_potrf32_s<kLS>(Sd, col, cbar, lane);
}

// The rows below the diagonal block, factored along with it (the panel TRSM of the
// reference's column loop, solver.cpp:21-33, on rows > the block): lane i owns one
// row's 32 panel entries at P; per column j, after warp_potrf32's arrival on cbar[j],
// l_i = a_ij * rsqrt(pivot_j) and a_ik -= l_i * l_kj for k > j.  The rsqrt repeats the
// diagonal warp's (same bits).  After a failed pivot the values are garbage, and the
// leaf is abandoned right after this phase (the abort flag).
__device__ __noinline__ void warp_tall32(double* P, const double* pub, uint64_t* cbar, uint32_t parity) {
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = P[c];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    mbar_wait(&cbar[j], parity);
    const double* cj = pub + (j + 1) * 40;  // column j's l values (and pivot j + 1)
    const double rj = rsqrt(pub[j * 40 + 32]);
    const double l = a[j] * rj;
    a[j] = l;
#pragma unroll
    for (int k = (j + 1) & ~1; k < 32; k += 2) {
      const double2 lk = *reinterpret_cast<const double2*>(cj + k);
      if (k > j) a[k] -= l * lk.x;
      if (k + 1 > j) a[k + 1] -= l * lk.y;
    }
  }
#pragma unroll
  for (int c = 0; c < 32; c += 2) *reinterpret_cast<double2*>(P + c) = make_double2(a[c], a[c + 1]);
}

// inverse of the lower 32x32 block at Sd into Db (row-major, stride kBS);
// lane c computes column c by forward substitution
template <int LS, int DS>
__device__ __noinline__ void warp_trtri32_s(const double* Sd, double* Db, int lane) {
  const double rinv = 1.0 / Sd[lane * LS + lane];  // lane i: 1 / L_ii, off the chain
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    double s0 = lane == i ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // 4 chains
#pragma unroll
    for (int k = 0; k < i; ++k) {
      const double t = Sd[i * LS + k] * x[k];
      if ((k & 3) == 0) s0 -= t;
      else if ((k & 3) == 1) s1 -= t;
      else if ((k & 3) == 2) s2 -= t;
      else s3 -= t;
    }
    const double ri = __shfl_sync(0xffffffffu, rinv, i);
    x[i] = i >= lane ? ((s0 + s1) + (s2 + s3)) * ri : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) Db[i * DS + lane] = x[i];
}
__device__ __forceinline__ void warp_trtri32(const double* Sd, double* Db, int lane) {
  warp_trtri32_s<kLS, kBS>(Sd, Db, lane);
}

#ifdef PKRR_LEAF_TRACE
__device__ long long g_leaf_trace[64];
// the __syncwarp keeps warp 0 converged (a lone-lane store left unreconverged would
// send every later __syncwarp / shuffle of the warp down its divergent path)
#define LEAF_MARK(i)                                   \
  {                                                    \
    if (threadIdx.x == 0) g_leaf_trace[i] = clock64(); \
    __syncwarp();                                      \
  }
#else
#define LEAF_MARK(i)
#endif

__global__ void __launch_bounds__(kLeafThreads, 1)
    potrf_leaf_kernel(double* __restrict__ A, int64_t lda, int kb, double* __restrict__ Linv,
                      int* status, int64_t m_valid, int factor, const double* __restrict__ fw = nullptr,
                      double* __restrict__ fz = nullptr) {
  pdl_wait();
  if (status && *reinterpret_cast<volatile int*>(status)) return;
  extern __shared__ double sm[];
  double* S = sm;                        // [128][132]: L (lower), X_ij^T in the upper blocks
  double* D = S + kNB * kLS;             // 4 x [32][36]: inv(L_bb)
  double* Tt = D + 4 * 32 * kBS;         // 3 x [32][36]: temporaries (transposed)
  uint64_t* lbar = reinterpret_cast<uint64_t*>(Tt + 3 * 32 * kBS);
  uint64_t* cbar = lbar + 1;  // [32] column j of the current panel published (warp_potrf32)
  uint64_t* dbar = cbar + 32; // [4] diagonal block pb factored
  int* flag = reinterpret_cast<int*>(dbar + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lr = lane >> 2, lk = lane & 3;
  const int64_t base = static_cast<int64_t>(kb) * kNB;
  double* Ab = A + base * lda + base;
  __shared__ double wsm[kNB];  // fused forward substitution: w_kb, final at kernel start
  if (fz && tid < kNB) wsm[tid] = fw[base + tid];
  // stage the 128 x 128 block: 128 row copies of 1 KB in flight at once (the
  // strict upper triangle is stale but never read as data)
  if (tid == 0) {
    *flag = 0;
    mbar_init(lbar, 1);
    for (int j = 0; j < 32; ++j) mbar_init(&cbar[j], 1);
    for (int j = 0; j < 4; ++j) mbar_init(&dbar[j], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(lbar, kNB * kNB * 8);
    for (int r = 0; r < kNB; ++r) bulk_load(S + r * kLS, Ab + static_cast<int64_t>(r) * lda, kNB * 8, lbar);
  }
  LEAF_MARK(0);
  __syncthreads();
  mbar_wait(lbar, 0);
  LEAF_MARK(1);

  if (!factor) {
    // diagonal-block inverses of a finished factor (launch_diag_inverses)
    if (warp < 4) warp_trtri32(S + (32 * warp) * kLS + 32 * warp, D + warp * 32 * kBS, lane);
  } else if (warp == 7) {
    // ---- warp 7: the 32x32 diagonal-block inverses, each as soon as its block is
    // factored, off the panel chain (they feed only the blocked inverse below) ----
    for (int pb = 0; pb < 4; ++pb) {
      mbar_wait(&dbar[pb], 0);
      if (*reinterpret_cast<volatile int*>(flag)) return;
      warp_trtri32(S + (32 * pb) * kLS + 32 * pb, D + pb * 32 * kBS, lane);
    }
  } else {
    // ---- warps 0-6: four 32-column panels.  Warp 0 factors the diagonal block,
    // warps 1..3-pb the rows below it in step (one column behind at most), then the
    // trailing SYRK inside the block; barriers among these 7 warps only ----
    for (int pb = 0; pb < 4; ++pb) {
      double* Sd = S + (32 * pb) * kLS + 32 * pb;
      const int R0 = 32 * (pb + 1);
      LEAF_MARK(2 + 5 * pb);
      if (warp == 0) {
        // Tt is free until the blocked inverse: two column buffers, then 32 published slots
        const int bad = warp_potrf32(Sd, Tt, cbar, lane);  // 33 column slots in Tt
#ifdef PKRR_LEAF_TRACE
        if (lane == 0) g_leaf_trace[40 + pb] = clock64();
        __syncwarp();
#endif
        if (bad >= 0 && lane == 0) {
          *flag = 1;
          if (status) {
            status[1] = static_cast<int>(base + 32 * pb + bad);
            __threadfence();
            atomicExch(&status[0], 1);
          }
        }
        __threadfence_block();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dbar[pb]);
      } else if (warp < 4 - pb) {
        warp_tall32(S + (R0 + 32 * (warp - 1) + lane) * kLS + 32 * pb, Tt, cbar, static_cast<uint32_t>(pb & 1));
#ifdef PKRR_LEAF_TRACE
        if (lane == 0) g_leaf_trace[44 + 4 * pb + warp] = clock64();
        __syncwarp();
#endif
      }
      consumer_sync(7 * 32);
      LEAF_MARK(3 + 5 * pb);
      if (*flag) return;
      if (pb == 3) break;
      // ---- trailing SYRK inside the block: S[R0:, R0:] -= P P^T over lower 16x16
      // blocks (2x2 DMMA tiles each; the upper tile of a diagonal block is not stored) ----
      const int nbt = (kNB - R0) / 16, nbl = nbt * (nbt + 1) / 2;
      for (int t = warp; t < nbl; t += 7) {
        int rb = 0;
        while ((rb + 1) * (rb + 2) / 2 <= t) ++rb;
        const int cb = t - rb * (rb + 1) / 2;
        double acc[2][2][2] = {};
        mma_2x2_rt(acc, S + (R0 + 16 * rb) * kLS + 32 * pb, S + (R0 + 16 * cb) * kLS + 32 * pb, kLS, 32, lr, lk);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (rb == cb && j > i) continue;
            double* dst = S + (R0 + 16 * rb + 8 * i + lr) * kLS + R0 + 16 * cb + 8 * j + 2 * lk;
            const double2 v = *reinterpret_cast<double2*>(dst);
            *reinterpret_cast<double2*>(dst) = make_double2(v.x - acc[i][j][0], v.y - acc[i][j][1]);
          }
      }
      consumer_sync(7 * 32);
      LEAF_MARK(4 + 5 * pb);
    }
    // L is final: its rows (lower part, 16-byte rounded -- the one extra column is a
    // zero of a diagonal 32-block) go out with plain vector stores while warp 7
    // finishes the last diagonal inverse; the blocked inverse below only writes S's
    // upper 32-blocks, beyond every stored row (fire-and-forget STG.128 drain while
    // the DMMAs run; the bulk-copy engine is slow for hundreds of small copies)
    for (int e = tid; e < kNB * 64; e += 7 * 32) {
      const int r = e >> 6, cp = e & 63;
      if (2 * cp <= r)
        *reinterpret_cast<double2*>(Ab + static_cast<int64_t>(r) * lda + 2 * cp) =
            *reinterpret_cast<const double2*>(S + r * kLS + 2 * cp);
    }
    LEAF_MARK(21);
  }
  // one barrier for every branch above (all warps reach this same call site)
  __syncthreads();

  LEAF_MARK(22);
  // ---- blocked inverse: X_ij = -D_i * sum_{k=j}^{i-1} L_ik X_kj, X_ij stored (not
  // transposed) in S's free upper block (j, i); T_j row-major in Tt[j].  Work item =
  // one 8-row tile x the 4 column tiles (the A fragment is loaded once per k step);
  // the lower-triangular D blocks bound the k ranges ----
  for (int bi = 1; bi < 4; ++bi) {
    for (int t = warp; t < bi * 4; t += 8) {
      const int bj = t >> 2, rt = t & 3;
      double acc[4][2] = {};
      const double* Arow = S + (32 * bi + 8 * rt) * kLS;
      mma_row4_rn_lowB(acc, Arow + 32 * bj, kLS, D + bj * 32 * kBS, kBS, lr, lk);  // X_jj = D_j
      for (int bk = bj + 1; bk < bi; ++bk)
        mma_row4_rn(acc, Arow + 32 * bk, kLS, S + (32 * bj) * kLS + 32 * bk, kLS, 0, 32, lr, lk);
      double* T = Tt + bj * 32 * kBS + (8 * rt + lr) * kBS + 2 * lk;
#pragma unroll
      for (int c = 0; c < 4; ++c) *reinterpret_cast<double2*>(T + 8 * c) = make_double2(acc[c][0], acc[c][1]);
    }
    __syncthreads();
    for (int t = warp; t < bi * 4; t += 8) {
      const int bj = t >> 2, rt = t & 3;
      double acc[4][2] = {};
      // row tile rt of the lower-triangular D_i has nonzeros in k < 8 rt + 8 only
      mma_row4_rn(acc, D + bi * 32 * kBS + (8 * rt) * kBS, kBS, Tt + bj * 32 * kBS, kBS, 0, 8 * rt + 8, lr, lk);
      double* X = S + (32 * bj + 8 * rt + lr) * kLS + 32 * bi + 2 * lk;
#pragma unroll
      for (int c = 0; c < 4; ++c) *reinterpret_cast<double2*>(X + 8 * c) = make_double2(-acc[c][0], -acc[c][1]);
    }
    __syncthreads();
  }

  LEAF_MARK(23);
  if (fz) {
    // fused forward substitution (see launch_potrf): z_kb = inv(L_kk) w_kb, w_kb being
    // final (every earlier panel's TRSM has subtracted its part); row i of inv(L_kk):
    // diagonal 32-block from D, the others from the X blocks in S's upper half
    if (tid < kNB) {
      const int bi = tid >> 5, r = tid & 31;
      double z0 = 0.0, z1 = 0.0, z2 = 0.0, z3 = 0.0;
      for (int bj = 0; bj <= bi; ++bj) {
        const double* src = bi == bj ? D + bi * 32 * kBS + r * kBS : S + (32 * bj + r) * kLS + 32 * bi;
        const double* wk = wsm + 32 * bj;
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          z0 = fma(src[c], wk[c], z0);
          z1 = fma(src[c + 1], wk[c + 1], z1);
          z2 = fma(src[c + 2], wk[c + 2], z2);
          z3 = fma(src[c + 3], wk[c + 3], z3);
        }
      }
      fz[base + tid] = (z0 + z1) + (z2 + z3);
    }
  }
  // the 10 lower 32x32 blocks of inv(L), 16 double2 per row segment (the upper blocks
  // of the Linv scratch are zeroed once at allocation)
  double* Lo = Linv + base * kNB;
  for (int e = tid; e < 10 * 32 * 16; e += kLeafThreads) {
    const int q = e >> 4, cp = e & 15;
    const int blk = q >> 5, r = q & 31;
    const int bi = blk < 1 ? 0 : (blk < 3 ? 1 : (blk < 6 ? 2 : 3));
    const int bj = blk - bi * (bi + 1) / 2;
    const double* src = bi == bj ? D + bi * 32 * kBS + r * kBS : S + (32 * bj + r) * kLS + 32 * bi;
    *reinterpret_cast<double2*>(Lo + (32 * bi + r) * kNB + 32 * bj + 2 * cp) =
        *reinterpret_cast<const double2*>(src + 2 * cp);
  }
  LEAF_MARK(24);
}


}  // namespace pk
#include "potrf_df.cuh"
namespace pk {

// ---------------------------------------------------------------------------
// dataflow Cholesky (potrf_df.cuh): the static task list and the launcher
// ---------------------------------------------------------------------------
namespace {
struct DfNode {
  int type;  // -1 chain step, else DfType
  int i, j, a, b, time, deadline;
  std::vector<int> out;
  int indeg;
};
}  // namespace

// Topological order of the worker tasks of an nt-tile factorization, the chain steps as
// virtual nodes processed as soon as they are ready (so every task a chain step waits
// on precedes every task that waits on that step), ties by deadline: the step by which
// the task's output is needed.
int df_band() {
  static const int d = std::getenv("PKRR_DF_BAND") ? std::atoi(std::getenv("PKRR_DF_BAND")) : 1 << 20;
  return d;
}
std::vector<int4> df_build_tasks(int nt, bool gram) {
  std::vector<DfNode> nd;
  auto add = [&](int type, int i, int j, int a, int b, int time) {
    nd.push_back(DfNode{type, i, j, a, b, time, 0, {}, 0});
    return static_cast<int>(nd.size()) - 1;
  };
  auto edge = [&](int from, int to) {
    nd[from].out.push_back(to);
    ++nd[to].indeg;
  };
  std::vector<int> chain(nt), trsm(static_cast<size_t>(nt) * nt, -1);
  std::vector<std::vector<int>> items(static_cast<size_t>(nt) * nt);
  for (int k = 0; k < nt; ++k) chain[k] = add(-1, k, k, 0, 0, k);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j <= i; ++j) {
      const int e = i == j ? j - 1 : j;  // panels [0, e) applied by workers (the chain applies j-1 to (j,j))
      if (e <= 0) continue;
      // the last kDfSingles panels singly (ready a step after their panel) only within
      // df_band() tile rows of the diagonal; farther tiles take the remainder as one batch
      const int s0 = std::max(0, e - (i - j <= df_band() ? kDfSingles : 0));
      std::vector<std::pair<int, int>> rng;
      // batch boundaries staggered per tile: aligned ones made every far tile's batch
      // come due on the same step (multiples of 8), queueing ~1000 K = 512 tasks ahead
      // of the single updates that step's chain work needed
      for (int a = 0; a < s0;) {
        const int len = a == 0 ? 1 + (i + j) % kDfBatch : kDfBatch;
        rng.push_back({a, std::min(a + len, s0)});
        a += len;
      }
      for (int q = s0; q < e; ++q) rng.push_back({q, q + 1});
      for (auto& r : rng) items[i * nt + j].push_back(add(DF_UPD, i, j, r.first, r.second, r.second - 1));
    }
  for (int k = 0; k < nt; ++k)
    for (int i = k + 2; i < nt; ++i) trsm[i * nt + k] = add(DF_TRSM, i, k, 0, 0, k);
  std::vector<int> inv;
  for (int b = 0; b < nt / 2; ++b) inv.push_back(add(DF_INV, b, 0, 0, 0, 2 * b + 1));
  // fused kernel-matrix build: GRAM(i, j) precedes everything that touches tile (i, j)
  std::vector<int> gramt(static_cast<size_t>(nt) * nt, -1);
  if (gram)
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j <= i; ++j) gramt[i * nt + j] = add(DF_GRAM, i, j, 0, 0, -1);
  auto lprod = [&](int row, int q) { return row == q + 1 ? chain[q] : trsm[row * nt + q]; };
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j <= i; ++j) {
      const std::vector<int>& it = items[i * nt + j];
      for (size_t x = 0; x < it.size(); ++x) {
        const int id = it[x];
        if (x > 0) edge(it[x - 1], id);
        const int q = nd[id].b - 1;
        edge(lprod(i, q), id);
        if (j != i) edge(lprod(j, q), id);
        nd[id].deadline = x + 1 < it.size() ? nd[it[x + 1]].time : (i == j ? j - 1 : j);
      }
    }
  for (int k = 0; k < nt; ++k)
    for (int i = k + 2; i < nt; ++i) {
      const int id = trsm[i * nt + k];
      edge(chain[k], id);
      if (!items[i * nt + k].empty()) edge(items[i * nt + k].back(), id);
      nd[id].deadline = k + 1;
    }
  for (int k = 0; k < nt; ++k) {
    if (k > 0) edge(chain[k - 1], chain[k]);
    if (!items[k * nt + k].empty()) edge(items[k * nt + k].back(), chain[k]);
    if (k + 1 < nt && !items[(k + 1) * nt + k].empty()) edge(items[(k + 1) * nt + k].back(), chain[k]);
  }
  if (gram)
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j <= i; ++j) {
        const int g = gramt[i * nt + j];
        const std::vector<int>& it = items[i * nt + j];
        if (!it.empty()) {
          // one step ahead of the tile's first update, not at its earliest start: early
          // keys queued ~2000 tile builds ahead of the first steps' critical tasks
          edge(g, it.front());
          nd[g].deadline = nd[it.front()].deadline - 1;
        } else if (i >= j + 2) {
          edge(g, trsm[i * nt + j]);
          nd[g].deadline = j;
        } else {
          edge(g, chain[j]);  // (j, j) or (j + 1, j): read by the chain at step j
          nd[g].deadline = j - 1;
        }
      }
  for (int b = 0; b < nt / 2; ++b) {
    edge(chain[2 * b + 1], inv[b]);
    nd[inv[b]].deadline = nt + 1;
  }
  using Key = std::tuple<int, int, int, int, int, int>;  // deadline, time, type, i, j, id
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> ready;
  std::vector<int> chain_ready;
  auto push = [&](int id) {
    if (nd[id].type < 0)
      chain_ready.push_back(id);
    else
      ready.push(Key{nd[id].deadline, nd[id].time, nd[id].type, nd[id].i, nd[id].j, id});
  };
  for (size_t id = 0; id < nd.size(); ++id)
    if (nd[id].indeg == 0) push(static_cast<int>(id));
  std::vector<int4> out;
  size_t done = 0;
  auto finish = [&](int id) {
    ++done;
    for (int o : nd[id].out)
      if (--nd[o].indeg == 0) push(o);
  };
  while (true) {
    while (!chain_ready.empty()) {
      const int id = chain_ready.back();
      chain_ready.pop_back();
      finish(id);
    }
    if (ready.empty()) break;
    const int id = std::get<5>(ready.top());
    ready.pop();
    const DfNode& n = nd[id];
    out.push_back(make_int4(n.type, n.i, n.j, n.a | (n.b << 16)));
    finish(id);
  }
  if (done != nd.size()) {
    fprintf(stderr, "pkrr: dataflow task graph has a cycle (%zu of %zu)\n", done, nd.size());
    abort();
  }
  return out;
}

// device copy of the task list per (device, nt), built once
static const int4* df_tasks_device(int nt, bool gram, int* ntasks) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, bool>, std::pair<int4*, int>> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(current_device(), nt, gram);
  auto it = cache.find(key);
  if (it == cache.end()) {
    const std::vector<int4> h = df_build_tasks(nt, gram);
    int4* d = nullptr;
    cudaMalloc(&d, sizeof(int4) * h.size());
    cudaMemcpy(d, h.data(), sizeof(int4) * h.size(), cudaMemcpyHostToDevice);
    it = cache.emplace(key, std::make_pair(d, static_cast<int>(h.size()))).first;
  }
  *ntasks = it->second.second;
  return it->second.first;
}

static bool launch_potrf_df(double* A, const CUtensorMap& tmA, double* Linv, int64_t mp, int* status, cudaStream_t s,
                            Counter& c, const FwdSolve* fs, const GramFuse* gf) {
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, potrf_df_kernel, kDfSmem);
  const int nt = static_cast<int>(mp / kDfT);
  DfParams p{};
  p.tasks = df_tasks_device(nt, gf != nullptr, &p.ntasks);
  const int64_t nflag = ((F_HEAD + static_cast<int64_t>(nt) * nt + nt + 2) + 31) / 32 * 32;
  const size_t bytes = nflag * 4 + sizeof(double) * (static_cast<size_t>(nt) * 4096 + static_cast<size_t>(nt) * nt * 64);
  // workspace: grow-only, one per (device, stream) -- calls on one stream are ordered,
  // so its previous use has finished; a per-call cudaMallocAsync / cudaFreeAsync made the
  // pool release and re-map the memory every call (~0.5 ms per C0 step)
  void* ws = nullptr;
  {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> pool;
    std::lock_guard<std::mutex> lock(mu);
    auto& e = pool[std::make_pair(current_device(), s)];
    if (e.second < bytes) {
      if (e.first) {
        cudaStreamSynchronize(s);
        cudaFree(e.first);
      }
      e.first = nullptr;
      e.second = 0;
      if (cudaMalloc(&e.first, bytes) == cudaSuccess) e.second = bytes;
    }
    ws = e.first;
  }
  cudaMemsetAsync(ws, 0, nflag * 4, s);
  p.flags = static_cast<int*>(ws);
  if (gf) {
    // tiles not yet formed: applied = -1 until their GRAM task
    cudaMemsetAsync(p.flags + F_HEAD, 0xff, sizeof(int) * static_cast<size_t>(nt) * nt, s);
    p.gram = 1;
    p.xk = static_cast<int>(gf->dp / kBK);
    p.m_valid = static_cast<int>(gf->m_valid);
    p.xnorm = gf->xnorm;
    p.K = gf->K;
    p.neg_inv_denom = -1.0 / ((2.0 * gf->sigma) * gf->sigma);
    p.shift = gf->shift;
  }
  p.inv64 = reinterpret_cast<double*>(p.flags + nflag);
  p.P = p.inv64 + static_cast<int64_t>(nt) * 4096;
  p.status = status ? status : p.flags + nflag - 2;
  p.A = A;
  p.lda = mp;
  p.nt = nt;
  p.Linv = Linv;
  p.y = fs ? fs->y : nullptr;
  p.z = fs ? fs->z : nullptr;
  CUtensorMap tmI;
  if (!make_tmap(&tmI, p.inv64, static_cast<int64_t>(nt) * kDfT, kDfT, kDfT)) {
    fprintf(stderr, "pkrr: tensor map for the dataflow Cholesky failed\n");
    abort();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(g_sms));
  cfg.blockDim = dim3(kDfThreads);
  cfg.dynamicSmemBytes = kDfSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const CUtensorMap tmX = gf ? gf->tmX : tmA;
  cudaLaunchKernelEx(&cfg, potrf_df_kernel, tmA, tmI, tmX, p);
  c.launched();
  return fs != nullptr;
}

// Panel-grouped blocked right-looking Cholesky.  G consecutive 128-column panels
// are factored with narrow column updates restricted to the group (leaf + DMMA
// TRSM each), then ONE trailing SYRK with K = 128*G updates the rest: the
// trailing matrix is streamed through HBM nb/G times instead of nb times.
static int g_panel_group = 0;  // 0: automatic (see launch_potrf)
// optional per-launch timing of the trailing SYRK (bench probe only)
static thread_local std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* g_syrk_events = nullptr;
static thread_local std::vector<double>* g_syrk_flops = nullptr;
void set_syrk_probe(std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* ev, std::vector<double>* fl) {
  g_syrk_events = ev;
  g_syrk_flops = fl;
}
static int g_syrk_persistent = 0;  // 0: one tile per CTA (priority-responsive); 1: one CTA per SM
static int g_syrk_ozaki = 0;       // 1: trailing SYRK on the int8 tensor cores (Ozaki splitting)

void set_panel_group(int g) { g_panel_group = g < 0 ? 0 : (g > 16 ? 16 : g); }
void set_syrk_persistent(int on) { g_syrk_persistent = on; }
void set_syrk_ozaki(int on) { g_syrk_ozaki = on; }
int syrk_ozaki() { return g_syrk_ozaki; }

// int8 slice tensor {K, R, 8} (K-contiguous), boxes {32, box_rows, 8}, 32B swizzle
static bool make_tmap_slices(CUtensorMap* m, const int8_t* base, int64_t R, int64_t K, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(R), 8};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(K * R)};
  cuuint32_t box[3] = {32u, static_cast<cuuint32_t>(box_rows), 8u};
  cuuint32_t es[3] = {1u, 1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- PKRR_SHADOW (debug): determinism checker for the factorisation steps ----
// Every step is run twice, on the live buffers and on copies taken just before it;
// a step whose output differs between the two runs depends on timing/concurrency.
// Each comparison records (max |diff|, count of differing elements) in a managed
// table; shadow_report() prints the differing steps and "N of M checks differ".
namespace {
constexpr int kShadowSlots = 1 << 16;
struct ShadowSlot {
  unsigned long long maxbits, count;
};
ShadowSlot* g_shadow = nullptr;
int g_shadow_n = 0;
std::vector<std::string> g_shadow_name;
}  // namespace

__global__ void shadow_diff_kernel(const double* A, const double* B, int64_t n, ShadowSlot* out) {
  double w = 0.0;
  unsigned long long cnt = 0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double a = A[e], b = B[e];
    if (a == b || (a != a && b != b)) continue;  // equal, or both NaN
    const double d = fabs(a - b);
    w = d > w ? d : w;
    ++cnt;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out->maxbits, static_cast<unsigned long long>(__double_as_longlong(w)));
    atomicAdd(&out->count, cnt);
  }
}

static void shadow_diff(const double* A, const double* B, int64_t n, cudaStream_t s, const std::string& name) {
  if (!g_shadow) {
    cudaMallocManaged(&g_shadow, sizeof(ShadowSlot) * kShadowSlots);
    memset(g_shadow, 0, sizeof(ShadowSlot) * kShadowSlots);
  }
  if (g_shadow_n >= kShadowSlots) return;
  g_shadow_name.push_back(name);
  shadow_diff_kernel<<<296, 256, 0, s>>>(A, B, n, g_shadow + g_shadow_n++);
}

void shadow_report() {
  if (!g_shadow) return;
  cudaDeviceSynchronize();
  int bad = 0;
  for (int i = 0; i < g_shadow_n; ++i) {
    if (g_shadow[i].count == 0) continue;
    ++bad;
    double w;
    memcpy(&w, &g_shadow[i].maxbits, 8);
    fprintf(stderr, "pkrr shadow: %s differs in %llu elements, max |diff| %.3e\n", g_shadow_name[i].c_str(),
            g_shadow[i].count, w);
  }
  fprintf(stderr, "pkrr shadow: %d of %d checks differ\n", bad, g_shadow_n);
  memset(g_shadow, 0, sizeof(ShadowSlot) * kShadowSlots);
  g_shadow_n = 0;
  g_shadow_name.clear();
}

namespace {
// the buffers one factorisation works on (the real ones, or the PKRR_SHADOW copies)
struct FactorBufs {
  double* A;
  CUtensorMap tmA;
  double* Linv;
  CUtensorMap tmLinv;
  int* status;
};
}  // namespace

bool potrf_df_eligible(int64_t mp, bool latency) {
  static const bool df_on = !(std::getenv("PKRR_DF") && std::atoi(std::getenv("PKRR_DF")) == 0);
  static const bool shadow = std::getenv("PKRR_SHADOW") != nullptr;
  return df_on && latency && mp / kNB < 64 && !shadow && !g_syrk_ozaki && g_panel_group == 0;
}

bool launch_potrf(double* A, const CUtensorMap& tmA, const CUtensorMap& tmLinv, double* Linv,
                  int64_t mp, int64_t m_valid, int* status, cudaStream_t s, Counter& c, int8_t* slices,
                  int* exps, cudaStream_t s2, bool latency, const FwdSolve* fs, const GramFuse* gf) {
  static std::atomic<uint64_t> attr_leaf{0}, attr_syrk{0}, attr_oz{0};
  smem_optin(attr_leaf, potrf_leaf_kernel, kLeafSmem);
  smem_optin(attr_syrk, dsyrk_persistent_kernel, kSyrkSmem);
  smem_optin(attr_oz, ozaki_syrk_kernel, kOzSmem);
  // Debug (PKRR_SHADOW): every step is run twice -- on A and on a copy taken just
  // before it -- and the two outputs compared (reported by shadow_report): a step
  // whose result depends on timing/concurrency shows up by name.
  static const bool shadow = std::getenv("PKRR_SHADOW") != nullptr;
  FactorBufs main{A, tmA, Linv, tmLinv, status}, sh{};
  if (shadow) {
    cudaMallocAsync(&sh.A, sizeof(double) * mp * mp, s);
    cudaMallocAsync(&sh.Linv, sizeof(double) * mp * kNB, s);
    if (status) {
      cudaMallocAsync(&sh.status, sizeof(int) * 8, s);
      cudaMemcpyAsync(sh.status, status, sizeof(int) * 2, cudaMemcpyDeviceToDevice, s);
    }
    make_tmap(&sh.tmA, sh.A, mp, mp, mp);
    make_tmap(&sh.tmLinv, sh.Linv, mp, kNB, kNB);
  }
  // a lone small system: the dataflow kernel (potrf_df.cuh); PKRR_DF=0 keeps the
  // stream-ordered panel chain below
  if (potrf_df_eligible(mp, latency)) return launch_potrf_df(A, tmA, Linv, mp, status, s, c, fs, gf);
  // fused forward substitution (not with the shadow checker: its steps run twice)
  const bool fused = fs != nullptr && !shadow;
  if (fused) cudaMemcpyAsync(fs->w, fs->y, sizeof(double) * mp, cudaMemcpyDeviceToDevice, s);
  int cur = 0;  // block index of the current step (shadow report tag)
  auto step = [&](const char* name, auto&& fn) {
    if (!shadow) {
      fn(main);
      return;
    }
    cudaMemcpyAsync(sh.A, A, sizeof(double) * mp * mp, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(sh.Linv, Linv, sizeof(double) * mp * kNB, cudaMemcpyDeviceToDevice, s);
    fn(main);
    fn(sh);
    const std::string tag = std::string(name) + " (mp " + std::to_string(mp) + ", block " + std::to_string(cur) + ")";
    shadow_diff(A, sh.A, mp * mp, s, tag);
    shadow_diff(Linv, sh.Linv, mp * kNB, s, tag + " Linv");
  };
  const int nb = static_cast<int>(mp / kNB);
  // leaf block of the recursive group blocking (panels whose column updates run as
  // column GEMMs; larger spans go through the SYRK kernel); PKRR_LEAF_BLOCK=2|8 measured
  // within 0.5% of 4 on C1 / C2
  static const int kLB = std::getenv("PKRR_LEAF_BLOCK") ? std::atoi(std::getenv("PKRR_LEAF_BLOCK")) : 4;
  // panels per trailing update: K = 512 for the int8 update and small systems (short
  // panel chains), K = 1024 from m >= 8192, K = 2048 from m >= 16384 (fewer passes over
  // the trailing matrix; the recursive blocking below keeps the intra-group work in
  // the SYRK kernel)
  const bool int8_update = g_syrk_ozaki && slices && exps;
  // A lone small system (latency-bound panel chain) uses G = 1: each panel's next
  // block column is updated at once by a 64-row-tile GEMM, the rest behind it.
  const int G = g_panel_group > 0 ? g_panel_group
                                  : (int8_update ? 4 : (nb < 64 ? (latency ? 1 : 4) : (nb < 128 ? 8 : 16)));
  // (a) of the trailing update (the next group's block columns) as a column GEMM with
  // 64-row tiles for narrow groups: K = 128 G is short, so spread it over more CTAs
  const bool gemm_a = G <= 2;
  // a lone system's panel steps (TRSM, next-column update) run on 32-row tiles: the
  // chain is latency-bound and twice the CTAs halve each CTA's share of the step
  const bool narrow_rows = latency && nb < 64;
  auto update_next = [&](const FactorBufs& f, int kb0_, int kend_, int G2, cudaStream_t st) {
    const int rem_ = nb - kend_;
    if (gemm_a) {
      GemmParams u{};
      u.a_row0 = u.b_row0 = kend_ * kNB;
      u.a_k0 = u.b_k0 = kb0_ * kNB;
      u.ktiles = (kend_ - kb0_) * (kNB / kBK);
      u.C = f.A;
      u.ldc = mp;
      u.c_row0 = u.c_col0 = kend_ * kNB;
      u.tiles_n = G2;
      u.abort_flag = f.status;
      if (narrow_rows) {
        u.tiles_m = 4 * rem_;
        gemm_launch<32, G_UPDATE>(f.tmA, f.tmA, u, u.tiles_m * G2, st, c);
      } else {
        u.tiles_m = 2 * rem_;
        gemm_launch<64, G_UPDATE>(f.tmA, f.tmA, u, u.tiles_m * G2, st, c);
      }
    } else {
      SyrkParams u{};
      u.row0 = kend_ * kNB;
      u.k0 = kb0_ * kNB;
      u.ktiles = (kend_ - kb0_) * (kNB / kBK);
      u.T = rem_;
      u.abort_flag = f.status;
      u.narrow = G2;
      dsyrk_persistent_kernel<<<syrk_tile_count(rem_, G2), kSyrkThreads, kSyrkSmem, st>>>(f.tmA, u);
      c.launched();
    }
  };
  // lookahead needs a second stream; not with the shadow checker or the int8 update
  const bool look = s2 != nullptr && !shadow && nb > 2 * G;
  cudaEvent_t ev_panel = nullptr, ev_b = nullptr;
  bool b_pending = false;
  if (look) {
    cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming);
  }
  for (int kb0 = 0; kb0 < nb; kb0 += G) {
    const int kend = kb0 + G < nb ? kb0 + G : nb;
    // Recursive blocking inside a group of G panels (leaf blocks of 4): when panel kb
    // starts the right child of a node of 2S panels (S >= 4), the left child's S panels
    // are applied to the right child's block columns in one narrow SYRK (K = 128 S);
    // column updates only span panels of the block's own leaf block of 4.  Every
    // (panel, block column) pair of the group is applied exactly once, most of them by
    // the SYRK kernel.
    for (int kb = kb0; kb < kend; ++kb) {
      const int off = kb - kb0;
      const int sub0 = kb0 + (off / kLB) * kLB;  // first panel of this block's leaf block
      for (int S = kLB; S < G; S *= 2) {
        if (off % (2 * S) != S) continue;
        cur = kb;
        step("half-update", [&](FactorBufs& f) {
          SyrkParams u{};
          u.row0 = kb * kNB;
          u.k0 = (kb - S) * kNB;
          u.ktiles = S * (kNB / kBK);
          u.T = nb - kb;
          u.abort_flag = f.status;
          u.narrow = std::min(S, kend - kb);
          dsyrk_persistent_kernel<<<syrk_tile_count(u.T, u.narrow), kSyrkThreads, kSyrkSmem, s>>>(f.tmA, u);
          c.launched();
        });
      }
      if (kb > sub0) {
        // column block kb (rows >= kb) -= A[:, sub0:kb] A[kb, sub0:kb]^T
        cur = kb;
        step("col-update", [&](FactorBufs& f) {
          GemmParams u{};
          u.a_row0 = kb * kNB;
          u.b_row0 = kb * kNB;
          u.a_k0 = u.b_k0 = sub0 * kNB;
          u.ktiles = (kb - sub0) * (kNB / kBK);
          u.C = f.A;
          u.ldc = mp;
          u.c_row0 = u.c_col0 = kb * kNB;
          u.tiles_n = 1;
          u.abort_flag = f.status;
          if (nb - kb < g_sms) {  // under one wave of 128-row tiles: 64-row tiles, twice the CTAs
            u.tiles_m = 2 * (nb - kb);
            gemm_launch<64, G_UPDATE>(f.tmA, f.tmA, u, u.tiles_m, s, c);
          } else {
            u.tiles_m = nb - kb;
            gemm_launch<128, G_UPDATE>(f.tmA, f.tmA, u, u.tiles_m, s, c);
          }
        });
      }
      cur = kb;
      step("leaf", [&](FactorBufs& f) {
        launch_pdl(potrf_leaf_kernel, 1, kLeafThreads, kLeafSmem, s, f.A, mp, kb, f.Linv, f.status, m_valid, 1,
                   fused ? static_cast<const double*>(fs->w) : nullptr, fused ? fs->z : nullptr);
        c.launched();
      });
      const int rem = nb - 1 - kb;
      if (rem <= 0) continue;
      // panel: A21 := A21 * inv(L11)^T  (in place, 64-row blocks)
      cur = kb;
      step("trsm", [&](FactorBufs& f) {
        GemmParams t{};
        t.a_row0 = (kb + 1) * kNB;
        t.a_k0 = kb * kNB;
        t.b_row0 = kb * kNB;
        t.b_k0 = 0;
        t.ktiles = kNB / kBK;
        t.C = f.A;
        t.ldc = mp;
        t.c_row0 = (kb + 1) * kNB;
        t.c_col0 = kb * kNB;
        t.tiles_n = 1;
        t.abort_flag = f.status;
        t.fz = fused ? fs->z + static_cast<int64_t>(kb) * kNB : nullptr;
        t.fw = fused ? fs->w : nullptr;
        if (narrow_rows) {
          t.tiles_m = rem * 4;
          gemm_launch<32, G_STORE>(f.tmA, f.tmLinv, t, rem * 4, s, c);
        } else {
          t.tiles_m = rem * 2;
          gemm_launch<64, G_STORE>(f.tmA, f.tmLinv, t, rem * 2, s, c);
        }
      });
    }
    const int rem = nb - kend;
    if (rem <= 0) continue;
    const int Kg = (kend - kb0) * kNB;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (g_syrk_events) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
    }
    cur = kend;
    if (int8_update && Kg == 512 && look) {
      // int8 update with lookahead: the group's panel rows are sliced once (into one of
      // two alternating slice buffers -- the previous group's (b) may still be reading
      // the other), (a) updates the next G2 block columns on s, (b) the rest on s2;
      // ordering as for the DMMA lookahead below.
      const int R = rem * kNB;
      const int buf = (kb0 / G) & 1;
      int8_t* sl = slices + static_cast<int64_t>(buf) * kOzS * mp * 512;
      int* ex = exps + static_cast<int64_t>(buf) * mp;
      ozaki_slice_kernel<<<(R * 32 + 255) / 256, 256, 0, s>>>(A, mp, kend * kNB, kb0 * kNB, R, Kg, sl, ex, status,
                                                              static_cast<int>(mp));
      CUtensorMap ta, tb;
      if (!make_tmap_slices(&ta, sl, mp, Kg, kOzM) || !make_tmap_slices(&tb, sl, mp, Kg, kOzN)) {
        fprintf(stderr, "pkrr: slice tensor map failed\n");
        abort();
      }
      const int G2 = rem < G ? rem : G;
      cudaEventRecord(ev_panel, s);  // panel and slices ready
      cudaStreamWaitEvent(s2, ev_panel, 0);
      if (b_pending) cudaStreamWaitEvent(s, ev_b, 0);
      OzParams op{};
      op.row0 = kend * kNB;
      op.R = R;
      op.ksteps = Kg / kOzK;
      op.exps = ex;
      op.abort_flag = status;
      op.srow = 0;
      op.narrow = G2 < rem ? 2 * G2 : 0;
      const int na = G2 < rem ? G2 * (G2 + 1) + (rem - G2) * 2 * G2 : rem * (rem + 1);
      ozaki_syrk_kernel<<<na, kOzThreads, kOzSmem, s>>>(ta, tb, tmA, op);
      c.launched(2);
      if (rem > G2) {
        OzParams ob = op;
        const int T2 = rem - G2;
        ob.row0 = (kend + G2) * kNB;
        ob.srow = G2 * kNB;
        ob.narrow = 0;
        ozaki_syrk_kernel<<<T2 * (T2 + 1), kOzThreads, kOzSmem, s2>>>(ta, tb, tmA, ob);
        c.launched();
        cudaEventRecord(ev_b, s2);
        b_pending = true;
      }
    } else if (int8_update && Kg == 512) {
      // int8 tensor-core trailing update (Ozaki splitting), FP64-accurate; fixed
      // geometry per part (slice stride mp rows) -> the same descriptors every group
      const int R = rem * kNB;
      step("int8-syrk", [&](FactorBufs& f) {
        ozaki_slice_kernel<<<(R * 32 + 255) / 256, 256, 0, s>>>(f.A, mp, kend * kNB, kb0 * kNB, R, Kg, slices,
                                                                exps, f.status, static_cast<int>(mp));
        CUtensorMap ta, tb;
        if (!make_tmap_slices(&ta, slices, mp, Kg, kOzM) || !make_tmap_slices(&tb, slices, mp, Kg, kOzN)) {
          fprintf(stderr, "pkrr: slice tensor map failed\n");
          abort();
        }
        OzParams op{};
        op.row0 = kend * kNB;
        op.R = R;
        op.ksteps = Kg / kOzK;
        op.exps = exps;
        op.abort_flag = f.status;
        ozaki_syrk_kernel<<<rem * (rem + 1), kOzThreads, kOzSmem, s>>>(ta, tb, f.tmA, op);
        c.launched(2);
      });
    } else if (look) {
      // lookahead: (a) the next panel's G tile columns now, on s, so the next panel
      // chain starts at once; (b) the rest of the trailing triangle on s2, overlapping
      // that chain.  Per tile the arithmetic is the full-update kernel's (same K order),
      // and (b) of this group runs after (b) of the previous one on s2, (a) after it too,
      // so every element sees the panels in the same order: bitwise the same factor.
      const int G2 = rem < G ? rem : G;
      if (b_pending) cudaStreamWaitEvent(s, ev_b, 0);
      if (!gemm_a) {
        cudaEventRecord(ev_panel, s);
        cudaStreamWaitEvent(s2, ev_panel, 0);
      }
      update_next(main, kb0, kend, G2, s);
      if (gemm_a) {
        // (b) behind (a): the short column GEMM gets the whole GPU (a persistent (b)
        // started first would leave it the reserved SMs only), (b) overlaps the next leaf
        cudaEventRecord(ev_panel, s);
        cudaStreamWaitEvent(s2, ev_panel, 0);
      }
      if (rem > G2) {
        SyrkParams v{};
        v.k0 = kb0 * kNB;
        v.ktiles = (kend - kb0) * (kNB / kBK);
        v.abort_flag = status;
        v.row0 = (kend + G2) * kNB;
        v.T = rem - G2;
        v.narrow = 0;
        // persistent grid on all but `reserve` SMs, so the (higher-priority) panel chain
        // always finds free SMs instead of waiting for a SYRK wave to drain
        static const int reserve = std::getenv("PKRR_LOOK_RESERVE") ? std::atoi(std::getenv("PKRR_LOOK_RESERVE")) : 8;
        const int nt = syrk_tile_count(v.T, 0);
        const int cap = g_sms - reserve;
        dsyrk_persistent_kernel<<<reserve > 0 && nt > cap ? cap : nt, kSyrkThreads, kSyrkSmem, s2>>>(tmA, v);
        c.launched();
        cudaEventRecord(ev_b, s2);
        b_pending = true;
      }
    } else {
      // trailing: A22 -= L21 L21^T over the whole group (K = 128 * group), C staged by TMA
      step("syrk", [&](FactorBufs& f) {
        if (gemm_a) {
          // same split as the lookahead path (bitwise-neutral): next columns, then the rest
          const int G2 = rem < G ? rem : G;
          update_next(f, kb0, kend, G2, s);
          if (rem == G2) return;
          SyrkParams v{};
          v.row0 = (kend + G2) * kNB;
          v.k0 = kb0 * kNB;
          v.ktiles = (kend - kb0) * (kNB / kBK);
          v.T = rem - G2;
          v.abort_flag = f.status;
          const int ntl = v.T * (v.T + 1) / 2;
          const int grid = g_syrk_persistent ? (ntl < g_sms ? ntl : g_sms) : ntl;
          dsyrk_persistent_kernel<<<grid, kSyrkThreads, kSyrkSmem, s>>>(f.tmA, v);
          c.launched();
          return;
        }
        SyrkParams u{};
        u.row0 = kend * kNB;
        u.k0 = kb0 * kNB;
        u.ktiles = (kend - kb0) * (kNB / kBK);
        u.T = rem;
        u.abort_flag = f.status;
        const int ntl = rem * (rem + 1) / 2;
        const int grid = g_syrk_persistent ? (ntl < g_sms ? ntl : g_sms) : ntl;
        dsyrk_persistent_kernel<<<grid, kSyrkThreads, kSyrkSmem, s>>>(f.tmA, u);
        c.launched();
      });
    }
    if (g_syrk_events) {
      cudaEventRecord(e1, s);
      g_syrk_events->push_back({e0, e1});
      // algorithmic: A22 -= L21 L21^T on the lower triangle incl. diagonal, K = 128*group
      const double rows = static_cast<double>(rem) * kNB;
      g_syrk_flops->push_back(rows * (rows + 1.0) * Kg);
    }
  }
  if (look) {
    if (b_pending) cudaStreamWaitEvent(s, ev_b, 0);
    cudaEventDestroy(ev_panel);  // destruction is deferred until the recorded work completes
    cudaEventDestroy(ev_b);
  }
  if (shadow) {
    cudaFreeAsync(sh.A, s);
    cudaFreeAsync(sh.Linv, s);
    if (sh.status) cudaFreeAsync(sh.status, s);
  }
  return fused;
}

void launch_diag_inverses(const double* L, int64_t mp, double* Linv, cudaStream_t s, Counter& c) {
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, potrf_leaf_kernel, kLeafSmem);
  const int nb = static_cast<int>(mp / kNB);
  for (int kb = 0; kb < nb; ++kb) {
    potrf_leaf_kernel<<<1, kLeafThreads, kLeafSmem, s>>>(const_cast<double*>(L), mp, kb, Linv,
                                                         nullptr, mp, 0);
    c.launched();
  }
}

__global__ void zero_upper_kernel(double* A, int64_t mp) {
  const int64_t total = mp * mp;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (e % mp > e / mp) A[e] = 0.0;
  }
}

void launch_zero_upper(double* A, int64_t mp, cudaStream_t s, Counter& c) {
  zero_upper_kernel<<<148 * 8, 256, 0, s>>>(A, mp);
  c.launched();
}

// ---------------------------------------------------------------------------
// blocked triangular solves with inter-CTA flags (ticket-ordered: CTA I only
// waits on blocks finished by CTAs that started before it -> no deadlock)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Both solves: CTA (ticket order) owns one 128-row block; thread (warp w, lane l)
// covers rows 16w..16w+15 x columns 4l..4l+3 of every 128x128 block it streams.
// A block's 16 row segments are loaded into registers BEFORE waiting for the flag
// of the vector block it multiplies, and partial sums stay per thread across all
// blocks (one cross-lane / cross-warp reduction per CTA), so the dependency chain
// costs one flag hand-off + one small diagonal-block product per step.
__device__ __forceinline__ double4 ldg_d4(const double* p) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ double4 ldcg_d4(const double* p) {
  const double2 a = __ldcg(reinterpret_cast<const double2*>(p)), b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void load_block16(const double* __restrict__ base, int64_t ld, double4 (&m)[16]) {
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) m[rr] = ldg_d4(base + rr * ld);
}
__device__ __forceinline__ void wait_flag(const int* f, int lane) {
  if (lane == 0)
    while (ld_acquire(f) == 0) {
    }
  __syncwarp();
}
__device__ __forceinline__ void prefetch_l2_block(const double* blk, int64_t ld, int tid) {
  // 128 rows x 1 KB: 1024 lines of 128 B, 4 per thread
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int line = tid + 256 * q, r = line >> 3, c = (line & 7) * 16;
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(blk + r * ld + c));
  }
}

// forward: z_I = inv(L_II) (b_I - sum_{K<I} L_IK z_K)
__global__ void __launch_bounds__(256) trsv_fwd_kernel(const double* __restrict__ L, int64_t ld,
                                                       const double* __restrict__ Linv,
                                                       const double* __restrict__ b, double* z,
                                                       int nb, int* ticket, int* flags,
                                                       const int* abort) {
  if (abort && *reinterpret_cast<const volatile int*>(abort)) return;
  __shared__ double sacc[kNB];
  __shared__ int sI;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  if (tid == 0) sI = atomicAdd(ticket, 1);
  __syncthreads();
  const int I = sI;
  prefetch_l2_block(Linv + static_cast<int64_t>(I) * kNB * kNB, kNB, tid);
  double bpre[16];  // b_I, loaded now: off the flag chain
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) bpre[rr] = lane == 0 ? __ldg(b + I * kNB + w * 16 + rr) : 0.0;
  const double* rows = L + (static_cast<int64_t>(I) * kNB + w * 16) * ld + lane * 4;
  double acc[16];
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) acc[rr] = 0.0;
  for (int K = 0; K < I; ++K) {
    double4 m[16];
    load_block16(rows + K * kNB, ld, m);
    wait_flag(&flags[K], lane);
    const double4 v = ldcg_d4(z + K * kNB + lane * 4);
#pragma unroll
    for (int rr = 0; rr < 16; ++rr)
      acc[rr] = fma(m[rr].w, v.w, fma(m[rr].z, v.z, fma(m[rr].y, v.y, fma(m[rr].x, v.x, acc[rr]))));
  }
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) {
    const double sum = warp_sum(acc[rr]);
    if (lane == 0) sacc[w * 16 + rr] = bpre[rr] - sum;
  }
  __syncthreads();
  const double4 v = *reinterpret_cast<const double4*>(sacc + lane * 4);
  double4 m[16];
  load_block16(Linv + (static_cast<int64_t>(I) * kNB + w * 16) * kNB + lane * 4, kNB, m);
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) {
    const double sum = warp_sum(fma(m[rr].w, v.w, fma(m[rr].z, v.z, fma(m[rr].y, v.y, m[rr].x * v.x))));
    if (lane == 0) z[I * kNB + w * 16 + rr] = sum;
  }
  __syncthreads();
  if (tid == 0) st_release(&flags[I], 1);
}

// backward: x_I = inv(L_II)^T (z_I - sum_{K>I} L_KI^T x_K)
__global__ void __launch_bounds__(256) trsv_bwd_kernel(const double* __restrict__ L, int64_t ld,
                                                       const double* __restrict__ Linv,
                                                       const double* __restrict__ z, double* x,
                                                       int nb, int* ticket, int* flags,
                                                       const int* abort, int ihi, unsigned long long* xt) {
  // xt != null: x blocks travel as tagged words (two 8-byte {32 data bits, tag} halves per
  // value, the tag set by the same store as the data: readers poll the data itself -- one
  // L2 round trip per chain step instead of flag, then data, and no fence before a flag);
  // xt == null: release / acquire flags (the distributed solve, whose later blocks are
  // final before the launch)
  if (abort && *reinterpret_cast<const volatile int*>(abort)) return;
  __shared__ double red[8][kNB];
  __shared__ double sv[kNB];
  __shared__ int sI;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  // blocks ihi-1, ihi-2, ... in ticket order (ihi = nb: the whole solve; the distributed
  // solve runs one super-column's blocks with the later x blocks already final)
  if (tid == 0) sI = ihi - 1 - atomicAdd(ticket, 1);
  __syncthreads();
  const int I = sI;
  // this thread's 16 x 4 piece of inv(L_II), parked in shared memory now (the same thread
  // reads it back): loading it after the last flag put an L2 round trip on every chain step
  extern __shared__ double4 sLinv[];
  {
    double4 m[16];
    load_block16(Linv + (static_cast<int64_t>(I) * kNB + w * 16) * kNB + lane * 4, kNB, m);
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) sLinv[rr * 256 + tid] = m[rr];
  }
  const double zI = tid < kNB ? __ldg(z + I * kNB + tid) : 0.0;  // z is final (previous kernel): load now
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // columns 4l..4l+3, partial over this warp's rows
  for (int K = nb - 1; K > I; --K) {
    double4 m[16];
    load_block16(L + (static_cast<int64_t>(K) * kNB + w * 16) * ld + I * kNB + lane * 4, ld, m);
    double xv = 0.0;
    if (xt) {
      const unsigned long long* src = xt + 2 * static_cast<int64_t>(K * kNB + w * 16 + (lane & 15));
      for (;;) {
        unsigned long long lo, hi;
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(lo), "=l"(hi) : "l"(src) : "memory");
        const bool ok = (lo >> 32) == 1ull && (hi >> 32) == 1ull;
        xv = __hiloint2double(static_cast<int>(hi & 0xffffffffull), static_cast<int>(lo & 0xffffffffull));
        if (__all_sync(0xffffffffu, ok)) break;
      }
    } else {
      wait_flag(&flags[K], lane);
      xv = lane < 16 ? __ldcg(x + K * kNB + w * 16 + lane) : 0.0;
    }
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
      const double v = __shfl_sync(0xffffffffu, xv, rr);
      a0 = fma(m[rr].x, v, a0);
      a1 = fma(m[rr].y, v, a1);
      a2 = fma(m[rr].z, v, a2);
      a3 = fma(m[rr].w, v, a3);
    }
  }
  *reinterpret_cast<double4*>(&red[w][lane * 4]) = make_double4(a0, a1, a2, a3);
  __syncthreads();
  if (tid < kNB) {
    double sum = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) sum += red[q][tid];
    sv[tid] = zI - sum;
  }
  __syncthreads();
  // x_I = Linv_I^T sv: column sums over this warp's 16 rows, then across warps
  a0 = a1 = a2 = a3 = 0.0;
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) {
    const double v = sv[w * 16 + rr];
    const double4 m = sLinv[rr * 256 + tid];
    a0 = fma(m.x, v, a0);
    a1 = fma(m.y, v, a1);
    a2 = fma(m.z, v, a2);
    a3 = fma(m.w, v, a3);
  }
  __syncthreads();
  *reinterpret_cast<double4*>(&red[w][lane * 4]) = make_double4(a0, a1, a2, a3);
  __syncthreads();
  if (tid < kNB) {
    double sum = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) sum += red[q][tid];
    x[I * kNB + tid] = sum;
    if (xt) {
      const unsigned long long lo = static_cast<unsigned int>(__double2loint(sum)) | (1ull << 32);
      const unsigned long long hi = static_cast<unsigned int>(__double2hiint(sum)) | (1ull << 32);
      asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};\n" ::"l"(xt + 2 * static_cast<int64_t>(I * kNB + tid)),
                   "l"(lo), "l"(hi)
                   : "memory");
    }
  }
  if (xt) return;
  __syncthreads();
  if (tid == 0) st_release(&flags[I], 1);  // st.release.gpu is the fence (no __threadfence before it)
}

// scratch of the solves: [2 nb + 2] tickets / flags, then (16-byte aligned) the tagged
// x words of the backward solve, 4 ints per row
size_t trsv_scratch_ints(int64_t mp) { return static_cast<size_t>((2 * (mp / kNB) + 2 + 3) / 4 * 4 + 4 * mp); }
static unsigned long long* trsv_tagged(int* scratch, int nb) {
  return reinterpret_cast<unsigned long long*>(scratch + (2 * nb + 2 + 3) / 4 * 4);
}
constexpr int kTrsvBwdSmem = 16 * 256 * 32;  // 128 KB: inv(L_II) in the threads' own slots
static void trsv_bwd_optin() {
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, trsv_bwd_kernel, kTrsvBwdSmem);
}

void launch_trsv_bwd(const double* L, const double* Linv, int64_t mp, const double* z, double* x,
                     int* scratch, const int* abort, cudaStream_t s, Counter& c) {
  const int nb = static_cast<int>(mp / kNB);
  cudaMemsetAsync(scratch, 0, sizeof(int) * trsv_scratch_ints(mp), s);
  trsv_bwd_optin();
  trsv_bwd_kernel<<<nb, 256, kTrsvBwdSmem, s>>>(L, mp, Linv, z, x, nb, scratch + 1, scratch + 2 + nb, abort, nb,
                                                trsv_tagged(scratch, nb));
  c.launched();
}

void launch_trsv(const double* L, const double* Linv, int64_t mp, const double* b, double* z,
                 double* x, int* scratch, const int* abort, cudaStream_t s, Counter& c) {
  const int nb = static_cast<int>(mp / kNB);
  cudaMemsetAsync(scratch, 0, sizeof(int) * trsv_scratch_ints(mp), s);
  trsv_bwd_optin();
  trsv_fwd_kernel<<<nb, 256, 0, s>>>(L, mp, Linv, b, z, nb, scratch, scratch + 2, abort);
  trsv_bwd_kernel<<<nb, 256, kTrsvBwdSmem, s>>>(L, mp, Linv, z, x, nb, scratch + 1, scratch + 2 + nb, abort, nb,
                                                trsv_tagged(scratch, nb));
  c.launched(2);
}

// ---------------------------------------------------------------------------
// assemble / GEMV / reductions
// ---------------------------------------------------------------------------
__global__ void assemble_kernel(const double2* __restrict__ K, double2* __restrict__ A, int64_t mp,
                                double shift, const int* abort, int lower) {
  if (abort && *reinterpret_cast<const volatile int*>(abort)) return;
  const int64_t total = mp * mp / 2;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = (2 * e) / mp, col = (2 * e) % mp;
    if (lower && col > r) continue;  // the factorization reads the lower triangle only
    double2 v = K[e];
    if (col == r) v.x += shift;
    if (col + 1 == r) v.y += shift;
    A[e] = v;
  }
}

void launch_assemble(const double* K, double* A, int64_t mp, double shift, const int* abort,
                     cudaStream_t s, Counter& c, bool lower_only) {
  assemble_kernel<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const double2*>(K),
                                         reinterpret_cast<double2*>(A), mp, shift, abort, lower_only ? 1 : 0);
  c.launched();
}

// y = K alpha for a symmetric K of which only the lower 128x128 tiles are stored (the
// pipeline's gram): CTA I streams its row tiles (I, J < I), the lower half of (I, I) and
// its column tiles (J > I, I) -- T tiles per CTA, balanced -- with per-thread partials
// (16 rows x 4 columns per thread, as in the triangular solves) reduced once, in a fixed
// order: deterministic.  alpha's padding entries are 0.
__global__ void __launch_bounds__(256) symv_lower_kernel(const double* __restrict__ K, int64_t ld, int nb,
                                                         const double* __restrict__ alpha, double* __restrict__ y,
                                                         const int* abort) {
  if (abort && *reinterpret_cast<const volatile int*>(abort)) return;
  __shared__ double red[8][kNB];
  __shared__ double yrow[kNB];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int I = blockIdx.x;
  // this CTA's share of the tile range (blockIdx.y of kSymvSplit): a partial y_I
  const int J0 = static_cast<int>(blockIdx.y) * nb / kSymvSplit;
  const int J1 = (static_cast<int>(blockIdx.y) + 1) * nb / kSymvSplit;
  y += static_cast<int64_t>(blockIdx.y) * nb * kNB;
  double ar[16];
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) ar[rr] = 0.0;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  const int64_t r0 = static_cast<int64_t>(I) * kNB + w * 16;
  for (int J = J0; J < (I < J1 ? I : J1); ++J) {  // row part: full tiles left of the diagonal
    double4 m[16];
    load_block16(K + r0 * ld + J * kNB + lane * 4, ld, m);
    const double4 v = ldg_d4(alpha + J * kNB + lane * 4);
#pragma unroll
    for (int rr = 0; rr < 16; ++rr)
      ar[rr] = fma(m[rr].w, v.w, fma(m[rr].z, v.z, fma(m[rr].y, v.y, fma(m[rr].x, v.x, ar[rr]))));
  }
  if (I >= J0 && I < J1) {  // diagonal tile: (r, c) with c <= r stands for itself and, if c < r, for (c, r)
    double4 m[16];
    load_block16(K + r0 * ld + I * kNB + lane * 4, ld, m);
    const double4 v = ldg_d4(alpha + I * kNB + lane * 4);
    const double xr = lane < 16 ? __ldg(alpha + r0 + lane) : 0.0;
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
      const int r = w * 16 + rr, c = lane * 4;
      const double xa = __shfl_sync(0xffffffffu, xr, rr);
      const double e0 = c <= r ? m[rr].x : 0.0, e1 = c + 1 <= r ? m[rr].y : 0.0;
      const double e2 = c + 2 <= r ? m[rr].z : 0.0, e3 = c + 3 <= r ? m[rr].w : 0.0;
      ar[rr] = fma(e3, v.w, fma(e2, v.z, fma(e1, v.y, fma(e0, v.x, ar[rr]))));
      c0 = fma(c < r ? m[rr].x : 0.0, xa, c0);
      c1 = fma(c + 1 < r ? m[rr].y : 0.0, xa, c1);
      c2 = fma(c + 2 < r ? m[rr].z : 0.0, xa, c2);
      c3 = fma(c + 3 < r ? m[rr].w : 0.0, xa, c3);
    }
  }
  for (int J = (I + 1 > J0 ? I + 1 : J0); J < J1; ++J) {  // column part: tiles below the diagonal, transposed
    double4 m[16];
    const int64_t rj = static_cast<int64_t>(J) * kNB + w * 16;
    load_block16(K + rj * ld + I * kNB + lane * 4, ld, m);
    const double xr = lane < 16 ? __ldg(alpha + rj + lane) : 0.0;
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) {
      const double xa = __shfl_sync(0xffffffffu, xr, rr);
      c0 = fma(m[rr].x, xa, c0);
      c1 = fma(m[rr].y, xa, c1);
      c2 = fma(m[rr].z, xa, c2);
      c3 = fma(m[rr].w, xa, c3);
    }
  }
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) {
    const double sum = warp_sum(ar[rr]);
    if (lane == 0) yrow[w * 16 + rr] = sum;
  }
  *reinterpret_cast<double4*>(&red[w][lane * 4]) = make_double4(c0, c1, c2, c3);
  __syncthreads();
  if (tid < kNB) {
    double sum = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) sum += red[q][tid];
    y[static_cast<int64_t>(I) * kNB + tid] = yrow[tid] + sum;
  }
}

void launch_symv_lower(const double* K, int64_t mp, const double* alpha, double* y, const int* abort,
                       cudaStream_t s, Counter& c) {
  const dim3 grid(static_cast<unsigned>(mp / kNB), kSymvSplit);
  symv_lower_kernel<<<grid, 256, 0, s>>>(K, mp, static_cast<int>(mp / kNB), alpha, y, abort);
  c.launched();
}

__global__ void __launch_bounds__(256) gemv_rows_kernel(const double* __restrict__ M, int64_t ld,
                                                        int64_t rows, int64_t cols,
                                                        const double* __restrict__ v,
                                                        double* __restrict__ out, const int* abort) {
  if (abort && *reinterpret_cast<const volatile int*>(abort)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  if (i >= rows) return;
  const double* row = M + i * ld;
  double s = 0.0;
  for (int64_t j = lane; j < cols; j += 32) s += row[j] * v[j];
  s = warp_sum(s);
  if (lane == 0) out[i] = s;
}

void launch_gemv_rows(const double* M, int64_t ld, int64_t rows, int64_t cols, const double* v,
                      double* out, const int* abort, cudaStream_t s, Counter& c) {
  if (rows <= 0) return;
  gemv_rows_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(M, ld, rows, cols, v, out,
                                                                        abort);
  c.launched();
}

// fixed-shape block tree reduction (deterministic)
__device__ double block_sum_1024(double v, double* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;  // valid in warp 0
}

__global__ void __launch_bounds__(1024) residual_finish_kernel(const double* __restrict__ Ka,
                                                               const double* __restrict__ alpha,
                                                               const double* __restrict__ y,
                                                               int64_t m, int64_t mp, double shift,
                                                               double* out, const int* abort) {
  if (abort && *reinterpret_cast<const volatile int*>(abort)) return;
  __shared__ double red[32];
  double rs = 0.0, ys = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    double ka = Ka[i];  // the symmetric GEMV's partial vectors, summed in a fixed order
#pragma unroll
    for (int q = 1; q < kSymvSplit; ++q) ka += Ka[q * mp + i];
    const double acc = (shift * alpha[i] - y[i]) + ka;
    rs += acc * acc;
    ys += y[i] * y[i];
  }
  const double R = block_sum_1024(rs, red);
  const double Y = block_sum_1024(ys, red);
  if (threadIdx.x == 0) {
    out[0] = Y > 0.0 ? sqrt(R / Y) : sqrt(R);
    out[1] = Y > 0.0 ? sqrt(R) / sqrt(Y) : sqrt(R);
  }
}

void launch_residual_finish(const double* Kalpha, const double* alpha, const double* y, int64_t m,
                            double shift, double* out, const int* abort, cudaStream_t s,
                            Counter& c) {
  const int64_t mp = (m + kNB - 1) / kNB * kNB;
  residual_finish_kernel<<<1, 1024, 0, s>>>(Kalpha, alpha, y, m, mp, shift, out, abort);
  c.launched();
}

__global__ void __launch_bounds__(1024) sse_scatter_kernel(const double* __restrict__ pred,
                                                           const int64_t* __restrict__ pos,
                                                           int64_t cnt,
                                                           const double* __restrict__ ytest,
                                                           double* pred_all, double* out,
                                                           const int* abort) {
  if (abort && *reinterpret_cast<const volatile int*>(abort)) return;
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < cnt; j += blockDim.x) {
    const double v = pred[j];
    const int64_t g = pos[j];
    if (pred_all) pred_all[g] = v;
    const double diff = v - ytest[g];
    s += diff * diff;
  }
  const double S = block_sum_1024(s, red);
  if (threadIdx.x == 0) out[0] = S;
}

void launch_sse_scatter(const double* pred, const int64_t* pos, int64_t cnt, const double* ytest,
                        double* pred_all, double* out, const int* abort, cudaStream_t s,
                        Counter& c) {
  sse_scatter_kernel<<<1, 1024, 0, s>>>(pred, pos, cnt, ytest, pred_all, out, abort);
  c.launched();
}

// predictor: 0 whole, 1 average, 2 nearest, 3 oracle (strategies.cpp:458-495)
__global__ void __launch_bounds__(1024) combine_kernel(const double* __restrict__ pp, int64_t p,
                                                       int64_t t, int predictor,
                                                       const int32_t* __restrict__ route,
                                                       const double* __restrict__ ytest,
                                                       double* pred, double* mse_out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < t; j += blockDim.x) {
    double v = 0.0;
    if (predictor == 0) {
      v = pp[j];
    } else if (predictor == 1) {
      for (int64_t q = 0; q < p; ++q) v += pp[q * t + j];
      v *= 1.0 / static_cast<double>(p);
    } else if (predictor == 2) {
      v = pp[static_cast<int64_t>(route[j]) * t + j];
    } else {
      double be = INFINITY;
      for (int64_t q = 0; q < p; ++q) {
        const double u = pp[q * t + j];
        const double err = (u - ytest[j]) * (u - ytest[j]);
        if (err < be) {
          be = err;
          v = u;
        }
      }
    }
    pred[j] = v;
    const double diff = v - ytest[j];
    s += diff * diff;
  }
  const double S = block_sum_1024(s, red);
  if (threadIdx.x == 0) mse_out[0] = S / static_cast<double>(t);
}

void launch_combine(const double* pp, int64_t p, int64_t t, int predictor, const int32_t* route,
                    const double* ytest, double* pred, double* mse_out, cudaStream_t s,
                    Counter& c) {
  combine_kernel<<<1, 1024, 0, s>>>(pp, p, t, predictor, route, ytest, pred, mse_out);
  c.launched();
}

// Cell combine + MSE of every cell at once (strategies.cpp:458-495 + mse :168-177).
// pp: per cell P x t predictions (P = 1: whole / nearest, already in test order; P = p:
// average / oracle, one row per part).  comb[cell][j] = the combined prediction;
// mse[cell] = sum_j (comb - y)^2 / t summed SEQUENTIALLY in test-row order with
// explicit round-to-nearest multiplies / adds (no FMA contraction): the arithmetic of
// the reference's mse(), so equal predictions give a bitwise equal MSE (and best cell).
// predictor 4: average by division (predict_average, strategies.cpp:135-140).
__global__ void combine_cells_kernel(const double* __restrict__ pp, int64_t P, int64_t t, int64_t ncell,
                                     int predictor, const double* __restrict__ y, double* __restrict__ comb) {
  const int64_t total = ncell * t;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / t, j = e % t;
    const double* base = pp + c * P * t;
    double v = 0.0;
    if (predictor == 0 || predictor == 2) {
      v = base[j];
    } else if (predictor == 1 || predictor == 4) {
      for (int64_t q = 0; q < P; ++q) v = __dadd_rn(v, base[q * t + j]);
      v = predictor == 1 ? __dmul_rn(v, 1.0 / static_cast<double>(P)) : __ddiv_rn(v, static_cast<double>(P));
    } else {
      double be = INFINITY;
      for (int64_t q = 0; q < P; ++q) {
        const double u = base[q * t + j];
        const double diff = __dsub_rn(u, y[j]);
        const double err = __dmul_rn(diff, diff);
        if (err < be) {
          be = err;
          v = u;
        }
      }
    }
    comb[e] = v;
  }
}

// One warp per cell: the lanes load 32 rows at a time (coalesced, the next 32 in flight)
// and form (pred - y)^2 with explicit roundings; lane 0 adds them in row order -- the
// reference's sequential sum, limited only by the dependent DADD latency.
__global__ void __launch_bounds__(32) mse_rows_kernel(const double* __restrict__ comb, const double* __restrict__ y,
                                                      int64_t t, double* __restrict__ mse) {
  const int64_t c = blockIdx.x;
  const int lane = threadIdx.x;
  const double* v = comb + c * t;
  double s = 0.0;
  auto sq = [&](int64_t j) {
    if (j >= t) return 0.0;
    const double diff = __dsub_rn(v[j], y[j]);
    return __dmul_rn(diff, diff);
  };
  double cur = sq(lane);
  for (int64_t base = 0; base < t; base += 32) {
    const double nxt = sq(base + 32 + lane);
    const int cnt = t - base < 32 ? static_cast<int>(t - base) : 32;
    for (int r = 0; r < cnt; ++r) {
      const double e = __shfl_sync(0xffffffffu, cur, r);
      s = __dadd_rn(s, e);
    }
    cur = nxt;
  }
  if (lane == 0) mse[c] = __ddiv_rn(s, static_cast<double>(t));
}

void launch_combine_cells(const double* pp, int64_t P, int64_t t, int64_t ncell, int predictor, const double* y,
                          double* comb, double* mse, cudaStream_t s, Counter& c) {
  if (t <= 0 || ncell <= 0) return;
  int64_t blocks = (ncell * t + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  combine_cells_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(pp, P, t, ncell, predictor, y, comb);
  c.launched();
  if (mse) {
    mse_rows_kernel<<<static_cast<unsigned>(ncell), 32, 0, s>>>(comb, y, t, mse);
    c.launched();
  }
}

// ---------------------------------------------------------------------------
// clustering
// ---------------------------------------------------------------------------
constexpr int kAssignRows = 128;

// clustering.cpp:79-96 (assign) / :159-176 (k-balance scan step) / :182-195 (route)
template <int KP>
__global__ void __launch_bounds__(kAssignRows)
    assign_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                  const double* __restrict__ xnorm, const double* __restrict__ centers,
                  const double* __restrict__ cnorm, int k, int mode,
                  const uint8_t* __restrict__ open, int64_t row0, int32_t* label,
                  double* best_dist, unsigned long long* changed) {
  // feature chunk staged per step: 16 for 64 centres (static shared memory <= 48 KB)
  constexpr int CH = KP > 32 ? 16 : kChunk;
  __shared__ double xs[kAssignRows][CH + 1];
  __shared__ double cs[KP][CH + 1];
  const int64_t rbase = row0 + static_cast<int64_t>(blockIdx.x) * kAssignRows;
  const int64_t i = rbase + threadIdx.x;
  bool need = i < n;
  if (need && mode == 1) {
    const int cur = label[i];
    need = cur < 0 || !open[cur];
  }
  if (!__syncthreads_or(need)) return;
  double min_d = INFINITY;
  int min_j = mode == 0 ? 0 : -1;
  const double xn = need ? xnorm[i] : 0.0;
  for (int jb = 0; jb < k; jb += KP) {
    double dot[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) dot[q] = 0.0;
    for (int64_t c0 = 0; c0 < d; c0 += CH) {
      const int cw = static_cast<int>(d - c0 < CH ? d - c0 : CH);
      __syncthreads();
      {
        // all 32 staging loads of this thread in flight before the first store
        double v[CH];
        const int cc = threadIdx.x & (CH - 1), r0 = threadIdx.x / CH;
#pragma unroll
        for (int u = 0; u < CH; ++u) {
          const int64_t gr = rbase + r0 + u * (kAssignRows / CH);
          v[u] = (gr < n && cc < cw) ? __ldg(X + gr * d + c0 + cc) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < CH; ++u) xs[r0 + u * (kAssignRows / CH)][cc] = v[u];
      }
      for (int e = threadIdx.x; e < KP * CH; e += kAssignRows) {
        const int q = e / CH, cc = e % CH;
        cs[q][cc] = (jb + q < k && cc < cw) ? centers[static_cast<int64_t>(jb + q) * d + c0 + cc] : 0.0;
      }
      __syncthreads();
      if (need) {
        for (int cc = 0; cc < cw; ++cc) {
          const double x = xs[threadIdx.x][cc];
#pragma unroll
          for (int q = 0; q < KP; ++q) dot[q] = __dadd_rn(dot[q], __dmul_rn(x, cs[q][cc]));
        }
      }
    }
    if (need) {
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const int j = jb + q;
        if (j >= k) break;
        if (mode == 1 && !open[j]) continue;
        double dist = __dsub_rn(__dadd_rn(xn, cnorm[j]), __dmul_rn(2.0, dot[q]));
        if (dist < 0.0) dist = 0.0;
        if (dist < min_d) {
          min_d = dist;
          min_j = j;
        }
      }
    }
  }
  unsigned ch = 0;
  if (need) {
    if (mode == 0) {
      if (label[i] != min_j) {
        label[i] = min_j;
        ch = 1;
      }
      if (best_dist) best_dist[i] = min_d;
    } else {
      label[i] = min_j;
    }
  }
  if (changed) {
    const int cnt = __syncthreads_count(ch);
    if (threadIdx.x == 0 && cnt) atomicAdd(changed, static_cast<unsigned long long>(cnt));
  }
}

// Lloyd assign / routing (mode 0) with the rows streamed by the bulk-copy engine: a
// persistent CTA of 64 threads (one row each) walks 64-row tiles of X, each tile one
// contiguous cp.async.bulk (64 d doubles: rows are contiguous in row-major X) into a
// two-stage shared-memory ring, so the next tile's HBM read overlaps this tile's dot
// products.  Each thread reads its own row with 16-byte shared loads (row stride 8 d
// bytes: conflict-free wavefronts) and the centres by broadcast.  Arithmetic exactly
// assign_kernel's: sequential __dmul_rn / __dadd_rn in feature order, (xn + cn) - 2 dot,
// clamp, strict < (bitwise the reference's labels, clustering.cpp:79-96, 182-195).
constexpr int kBulkRows = 64, kBulkStages = 2;

// TPR threads per row: with 2, warps 0-1 take the first KP / 2 centres of the tile's 64 rows
// and warps 2-3 the rest (8 warps per SM instead of 4: one warp per scheduler left every
// barrier wait and LDS latency exposed); the halves' minima meet through shared memory,
// the lower half winning ties -- the sequential scan's strict < (clustering.cpp:79-96).
template <int KP, int TPR>
__global__ void __launch_bounds__(kBulkRows * TPR, 2)
    assign_bulk_kernel(const double* __restrict__ X, int64_t n, int d, const double* __restrict__ xnorm,
                       const double* __restrict__ centers, const double* __restrict__ cnorm, int k,
                       int64_t row0, int32_t* label, double* best_dist, unsigned long long* changed) {
  constexpr int KH = KP / TPR;  // centres per thread
  extern __shared__ __align__(16) unsigned char bulk_smem[];
  double* tiles = reinterpret_cast<double*>(bulk_smem);
  double* cs = tiles + kBulkStages * kBulkRows * d;  // [KP][d] centres (zero beyond k)
  __shared__ uint64_t full[kBulkStages + 1];  // + the centres' barrier
  __shared__ double cn_s[KP];
  __shared__ double hmin_d[kBulkRows];
  __shared__ int hmin_j[kBulkRows];
  const int tid = threadIdx.x;
  const int row = tid % kBulkRows, half = tid / kBulkRows;
  const int q0 = half * KH;
  const int64_t rows = n - row0;
  const int64_t ntiles = (rows + kBulkRows - 1) / kBulkRows;
  auto tile_bytes = [&](int64_t t) {
    const int64_t r = rows - t * kBulkRows;
    return static_cast<uint32_t>((r < kBulkRows ? r : kBulkRows) * d * 8);
  };
  if (tid == 0) {
    for (int s = 0; s <= kBulkStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    // the k centres (contiguous k d doubles) by one bulk copy, ahead of the first tile
    mbar_arrive_expect_tx(&full[kBulkStages], static_cast<uint32_t>(k * d * 8));
    bulk_load(cs, centers, static_cast<uint32_t>(k * d * 8), &full[kBulkStages]);
    for (int s = 0; s < kBulkStages; ++s) {
      const int64_t t = blockIdx.x + static_cast<int64_t>(s) * gridDim.x;
      if (t < ntiles) {
        mbar_arrive_expect_tx(&full[s], tile_bytes(t));
        bulk_load(tiles + s * kBulkRows * d, X + (row0 + t * kBulkRows) * d, tile_bytes(t), &full[s]);
      }
    }
  }
  for (int e = k * d + tid; e < KP * d; e += kBulkRows * TPR) cs[e] = 0.0;  // centres beyond k
  if (tid < KP) cn_s[tid] = tid < k ? cnorm[tid] : 0.0;
  __syncthreads();
  mbar_wait(&full[kBulkStages], 0);
  unsigned ch = 0;
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % kBulkStages;
    const int64_t i = row0 + t * kBulkRows + row;
    // the row's norm and label are read before waiting for its tile
    const double xn = i < n ? xnorm[i] : 0.0;
    const int lab = i < n && half == 0 ? label[i] : 0;
    mbar_wait(&full[s], static_cast<uint32_t>((it / kBulkStages) & 1));
    double min_d = INFINITY;
    int min_j = 0;
    if (i < n) {
      const double* xr = tiles + s * kBulkRows * d + row * d;
      double dot[KH];
#pragma unroll
      for (int q = 0; q < KH; ++q) dot[q] = 0.0;
      for (int c = 0; c < d; c += 2) {
        const double2 x = *reinterpret_cast<const double2*>(xr + c);
#pragma unroll
        for (int q = 0; q < KH; ++q) {
          const double2 cv = *reinterpret_cast<const double2*>(cs + (q0 + q) * d + c);
          dot[q] = __dadd_rn(dot[q], __dmul_rn(x.x, cv.x));
          dot[q] = __dadd_rn(dot[q], __dmul_rn(x.y, cv.y));
        }
      }
#pragma unroll
      for (int q = 0; q < KH; ++q) {
        if (q0 + q >= k) break;
        double dist = __dsub_rn(__dadd_rn(xn, cn_s[q0 + q]), __dmul_rn(2.0, dot[q]));
        if (dist < 0.0) dist = 0.0;
        if (dist < min_d) {
          min_d = dist;
          min_j = q0 + q;
        }
      }
    }
    if (TPR > 1) {
      if (half == 1) {
        hmin_d[row] = min_d;
        hmin_j[row] = min_j;
      }
      __syncthreads();
      if (half == 0 && hmin_d[row] < min_d) {  // strict: the lower centre index keeps a tie
        min_d = hmin_d[row];
        min_j = hmin_j[row];
      }
    }
    if (i < n && half == 0) {
      if (lab != min_j) {
        label[i] = min_j;
        ch += 1;
      }
      if (best_dist) best_dist[i] = min_d;
    }
    __syncthreads();  // every row of stage s consumed: refill it
    if (tid == 0) {
      const int64_t tn = t + static_cast<int64_t>(kBulkStages) * gridDim.x;
      if (tn < ntiles) {
        mbar_arrive_expect_tx(&full[s], tile_bytes(tn));
        bulk_load(tiles + s * kBulkRows * d, X + (row0 + tn * kBulkRows) * d, tile_bytes(tn), &full[s]);
      }
    }
  }
  if (changed) {
    const unsigned w = __reduce_add_sync(0xffffffffu, ch);
    if ((tid & 31) == 0 && w) atomicAdd(changed, static_cast<unsigned long long>(w));
  }
}

template <int KP, int TPR>
static bool try_assign_bulk_t(const double* X, int64_t n, int64_t d, const double* xnorm, const double* centers,
                              const double* cnorm, int k, int64_t row0, int32_t* label, double* best_dist,
                              unsigned long long* changed, cudaStream_t s, Counter& c) {
  const size_t smem = sizeof(double) * (static_cast<size_t>(kBulkStages) * kBulkRows * d + KP * d);
  if (d % 2 || (reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(centers) & 15) ||
      smem > 110 * 1024)
    return false;
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, assign_bulk_kernel<KP, TPR>, 110 * 1024);
  const int64_t ntiles = (n - row0 + kBulkRows - 1) / kBulkRows;
  const int64_t grid = ntiles < 2 * g_sms ? ntiles : 2 * g_sms;
  assign_bulk_kernel<KP, TPR><<<static_cast<unsigned>(grid), kBulkRows * TPR, smem, s>>>(
      X, n, static_cast<int>(d), xnorm, centers, cnorm, k, row0, label, best_dist, changed);
  c.launched();
  return true;
}
template <int KP>
static bool try_assign_bulk(const double* X, int64_t n, int64_t d, const double* xnorm, const double* centers,
                            const double* cnorm, int k, int64_t row0, int32_t* label, double* best_dist,
                            unsigned long long* changed, cudaStream_t s, Counter& c) {
  // two threads per row from 8 centres (PKRR_ASSIGN_TPR=1: one)
  static const int tpr = std::getenv("PKRR_ASSIGN_TPR") ? std::atoi(std::getenv("PKRR_ASSIGN_TPR")) : 2;
  if (KP >= 8 && tpr == 2)
    return try_assign_bulk_t<KP, (KP >= 8 ? 2 : 1)>(X, n, d, xnorm, centers, cnorm, k, row0, label, best_dist, changed,
                                                   s, c);
  return try_assign_bulk_t<KP, 1>(X, n, d, xnorm, centers, cnorm, k, row0, label, best_dist, changed, s, c);
}

// Lloyd assign / routing (mode 0) with a tensor-core distance SCREEN and an exact
// recompute -- bitwise the reference's labels and distances:
//  1. the CTA streams 64-row tiles of X by TMA (16-feature boxes, 128 B swizzle, zero
//     fill past d) through a two-stage ring; each warp computes its 32 rows' dot
//     products with all k centres by DMMA (m8n8k4 f64: ~1/8 of the FP64 issue of the
//     non-FMA dot products);
//  2. per row (one lane each): approximate distances a_q = max(0, (xn + cn_q) - 2 dot_q)
//     and a bound e_q = (4 d + 16) 2^-53 (xn + cn_q) >= |a_q - exact_q| (the DMMA and the
//     sequential dot each err by <= d u sum|x c| <= d u (xn + cn_q) / 2);
//  3. candidates = {q : a_q - e_q <= min_j (a_j + e_j)} -- every index that can reach the
//     exact minimum (ties included) and no other; their EXACT distances are recomputed
//     in the reference's arithmetic (sequential __dmul_rn / __dadd_rn over the features,
//     (xn + cn) - 2 dot, clamp) and the strict-< argmin in index order picks the winner.
// Usually one candidate per row, so the FP64 pipe does ~1/8 of assign_kernel's work and
// the kernel streams X at the memory rate.
constexpr int kSRows = 64, kSStages = 2;

template <int KP>
__global__ void __launch_bounds__(kSRows, KP <= 16 ? 2 : 1)
    assign_dmma_kernel(const __grid_constant__ CUtensorMap tmX, int64_t n, int d, const double* __restrict__ xnorm,
                       const double* __restrict__ centers, const double* __restrict__ cnorm, int k, int64_t row0,
                       int32_t* label, double* best_dist, unsigned long long* changed, double* debug) {
  extern __shared__ unsigned char sc_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(sc_smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int nch = (d + 15) / 16, dch = nch * 16, cstr = dch + 2;  // centre row stride (bank spread)
  const int stage_bytes = nch * 64 * 128;
  double* cs = reinterpret_cast<double*>(smem + kSStages * stage_bytes);  // [KP][cstr]
  double* dots = cs + KP * cstr;                                          // [kSRows][KP + 1]
  __shared__ uint64_t full[kSStages];
  __shared__ double cn_s[KP];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t rows = n - row0;
  const int64_t ntiles = (rows + kSRows - 1) / kSRows;
  auto issue = [&](int s, int64_t t) {
    mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(stage_bytes));
    for (int c = 0; c < nch; ++c)
      tma_load_2d(smem + s * stage_bytes + c * 64 * 128, &tmX, c * 16, static_cast<int>(row0 + t * kSRows), &full[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < kSStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    prefetch_tmap(&tmX);
    for (int s = 0; s < kSStages; ++s)
      if (blockIdx.x + static_cast<int64_t>(s) * gridDim.x < ntiles) issue(s, blockIdx.x + static_cast<int64_t>(s) * gridDim.x);
  }
  const uint32_t cbase = smem_u32(cs), dbase = smem_u32(dots);
  for (int e = tid; e < KP * cstr; e += kSRows) {
    const int q = e / cstr, f = e % cstr;
    sts_f64(cbase + 8u * e, (q < k && f < d) ? __ldg(centers + static_cast<int64_t>(q) * d + f) : 0.0);
  }
  if (tid < KP) cn_s[tid] = tid < k ? cnorm[tid] : 0.0;
  __syncthreads();
  const int lr = lane >> 2, lk = lane & 3;
  const double unit = 1.1102230246251565e-16;  // 2^-53
  const double ebound = (4.0 * d + 16.0) * unit;
  unsigned ch = 0;
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % kSStages;
    const int64_t i = row0 + t * kSRows + tid;  // this lane's row in the candidate phase
    const double xn = i < n ? xnorm[i] : 0.0;
    const int lab = i < n ? label[i] : 0;
    mbar_wait(&full[s], static_cast<uint32_t>((it / kSStages) & 1));
    const unsigned char* st = smem + s * stage_bytes;
    // ---- 1. DMMA screen: rows warp*32 + mt*8 + lr, centres nt*8 + 2 lk + e ----
    {
      double acc[4][KP / 8][2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < KP / 8; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
      for (int ks = 0; ks < dch / 4; ++ks) {
        const int kk = ks * 4 + lk;
        const unsigned char* chunk = st + (kk >> 4) * 64 * 128;
        double af[4], bf[KP / 8];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) af[mt] = lds_f64(chunk, swz128(warp * 32 + mt * 8 + lr, kk & 15));
#pragma unroll
        for (int nt = 0; nt < KP / 8; ++nt) bf[nt] = lds_f64_at(cbase + 8u * ((nt * 8 + lr) * cstr + kk));
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < KP / 8; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < KP / 8; ++nt) {
          const int r = warp * 32 + mt * 8 + lr, q = nt * 8 + 2 * lk;
          sts_f64(dbase + 8u * (r * (KP + 1) + q), acc[mt][nt][0]);
          sts_f64(dbase + 8u * (r * (KP + 1) + q + 1), acc[mt][nt][1]);
        }
    }
    __syncwarp();
    // ---- 2./3. candidates and their exact distances, one row per lane ----
    if (i < n) {
      double hi = INFINITY;
      for (int q = 0; q < k; ++q) {
        double a = (xn + cn_s[q]) - 2.0 * lds_f64_at(dbase + 8u * (tid * (KP + 1) + q));
        a = a < 0.0 ? 0.0 : a;
        const double e = ebound * (xn + cn_s[q]);
        hi = fmin(hi, a + e);
      }
      // candidates in index order, one per pass, every lane on its own next candidate
      // (the passes are warp-uniform: usually exactly one)
      double min_d = INFINITY;
      int min_j = 0, ncand = 0, q = -1;
      auto next_cand = [&](int from) {
        for (int r = from; r < k; ++r) {
          double a = (xn + cn_s[r]) - 2.0 * lds_f64_at(dbase + 8u * (tid * (KP + 1) + r));
          a = a < 0.0 ? 0.0 : a;
          if (a - ebound * (xn + cn_s[r]) <= hi) return r;
        }
        return -1;
      };
      q = next_cand(0);
      while (q >= 0) {
        ++ncand;
        double dot = 0.0;
        const uint32_t crow = cbase + 8u * (q * cstr);
        for (int f = 0; f < d; ++f) {
          const double x = lds_f64(st + (f >> 4) * 64 * 128, swz128(tid, f & 15));
          dot = __dadd_rn(dot, __dmul_rn(x, lds_f64_at(crow + 8u * f)));
        }
        double dist = __dsub_rn(__dadd_rn(xn, cn_s[q]), __dmul_rn(2.0, dot));
        if (dist < 0.0) dist = 0.0;
        if (dist < min_d) {
          min_d = dist;
          min_j = q;
        }
        q = next_cand(q + 1);
      }
      if (lab != min_j) {
        label[i] = min_j;
        ch += 1;
      }
      if (best_dist) best_dist[i] = min_d;
      if (debug) {  // PKRR_ASSIGN_DEBUG: candidates, the winner's screen error and bound
        debug[3 * (i - row0)] = ncand;
        const double a = (xn + cn_s[min_j]) - 2.0 * lds_f64_at(dbase + 8u * (tid * (KP + 1) + min_j));
        debug[3 * (i - row0) + 1] = (a < 0.0 ? 0.0 : a) - min_d;
        debug[3 * (i - row0) + 2] = ebound * (xn + cn_s[min_j]);
      }
    }
    __syncthreads();  // stage s (and the dot scratch) consumed: refill
    if (tid == 0 && t + static_cast<int64_t>(kSStages) * gridDim.x < ntiles)
      issue(s, t + static_cast<int64_t>(kSStages) * gridDim.x);
  }
  if (changed) {
    const unsigned w = __reduce_add_sync(0xffffffffu, ch);
    if (lane == 0 && w) atomicAdd(changed, static_cast<unsigned long long>(w));
  }
}

template <int KP>
static bool try_assign_dmma(const double* X, int64_t n, int64_t d, const double* xnorm, const double* centers,
                            const double* cnorm, int k, int64_t row0, int32_t* label, double* best_dist,
                            unsigned long long* changed, cudaStream_t s, Counter& c) {
  const int64_t nch = (d + 15) / 16, dch = nch * 16;
  const size_t smem = kSStages * nch * 64 * 128 + sizeof(double) * (KP * (dch + 2) + kSRows * (KP + 1)) + 1024;
  if (d % 2 || (reinterpret_cast<uintptr_t>(X) & 15) || smem > 200 * 1024) return false;
  CUtensorMap tm;
  if (!make_tmap(&tm, X, n, d, d)) return false;
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, assign_dmma_kernel<KP>, static_cast<int>(smem > 113 * 1024 ? smem : 113 * 1024));
  const int64_t ntiles = (n - row0 + kSRows - 1) / kSRows;
  const int per_sm = smem <= 113 * 1024 ? 2 : 1;
  const int64_t grid = ntiles < per_sm * g_sms ? ntiles : per_sm * g_sms;
  static double* debug = nullptr;
  static const bool dbg = std::getenv("PKRR_ASSIGN_DEBUG") != nullptr;
  if (dbg && !debug) cudaMallocManaged(&debug, sizeof(double) * 3 * (n - row0));
  assign_dmma_kernel<KP><<<static_cast<unsigned>(grid), kSRows, smem, s>>>(
      tm, n, static_cast<int>(d), xnorm, centers, cnorm, k, row0, label, best_dist, changed, debug);
  c.launched();
  if (dbg) {
    cudaStreamSynchronize(s);
    double mx = 0, err = 0, bound = 0;
    for (int64_t r = 0; r < n - row0; ++r) {
      mx += debug[3 * r];
      err = fmax(err, fabs(debug[3 * r + 1]));
      bound = fmax(bound, debug[3 * r + 2]);
    }
    fprintf(stderr, "assign_dmma: %.3f candidates per row, max |screen - exact| %.3e, max bound %.3e\n",
            mx / static_cast<double>(n - row0), err, bound);
  }
  return true;
}

void launch_assign(const double* X, int64_t n, int64_t d, const double* xnorm,
                   const double* centers, const double* cnorm, int k, int mode,
                   const uint8_t* open, int64_t row0, int32_t* label, double* best_dist,
                   unsigned long long* changed, cudaStream_t s, Counter& c) {
  const int64_t rows = n - row0;
  if (rows <= 0) return;
  // mode 0 (Lloyd assign, routing): bulk-copy row streaming (k-balance rounds, mode 1, skip
  // whole blocks of settled rows and keep the per-chunk kernel below)
  // 1 (default): bulk-copy streaming for k <= 16; 3: the DMMA screen (measured slower:
  // DESIGN.md); 0: the chunked kernel below for every k
  static const int variant = std::getenv("PKRR_ASSIGN") ? std::atoi(std::getenv("PKRR_ASSIGN")) : 1;
  if (mode == 0 && variant == 1) {
    if (k <= 8 && try_assign_bulk<8>(X, n, d, xnorm, centers, cnorm, k, row0, label, best_dist, changed, s, c))
      return;
    if (k > 8 && k <= 16 &&
        try_assign_bulk<16>(X, n, d, xnorm, centers, cnorm, k, row0, label, best_dist, changed, s, c))
      return;
  }
  if (mode == 0 && variant == 3) {
    if (k <= 8 && try_assign_dmma<8>(X, n, d, xnorm, centers, cnorm, k, row0, label, best_dist, changed, s, c))
      return;
    if (k > 8 && k <= 16 &&
        try_assign_dmma<16>(X, n, d, xnorm, centers, cnorm, k, row0, label, best_dist, changed, s, c))
      return;
    if (k > 16 && k <= 32 &&
        try_assign_dmma<32>(X, n, d, xnorm, centers, cnorm, k, row0, label, best_dist, changed, s, c))
      return;
    if (k > 32 && k <= 64 &&
        try_assign_dmma<64>(X, n, d, xnorm, centers, cnorm, k, row0, label, best_dist, changed, s, c))
      return;
  }
  const unsigned blocks = static_cast<unsigned>((rows + kAssignRows - 1) / kAssignRows);
  if (k <= 8)
    assign_kernel<8><<<blocks, kAssignRows, 0, s>>>(X, n, d, xnorm, centers, cnorm, k, mode, open,
                                                   row0, label, best_dist, changed);
  else if (k <= 16)
    assign_kernel<16><<<blocks, kAssignRows, 0, s>>>(X, n, d, xnorm, centers, cnorm, k, mode, open,
                                                    row0, label, best_dist, changed);
  else if (k <= 32)
    assign_kernel<32><<<blocks, kAssignRows, 0, s>>>(X, n, d, xnorm, centers, cnorm, k, mode, open,
                                                    row0, label, best_dist, changed);
  else  // one pass over X for up to 64 centres (the weak-scaled partitions: k = 8 per GPU)
    assign_kernel<64><<<blocks, kAssignRows, 0, s>>>(X, n, d, xnorm, centers, cnorm, k, mode, open,
                                                    row0, label, best_dist, changed);
  c.launched();
}

// ---- stable grouping: block counts -> scan -> scatter ----------------------
constexpr int kGroupRows = 256;

__global__ void group_count_kernel(const int32_t* __restrict__ label, int64_t n, int k,
                                   int64_t* counts) {
  extern __shared__ int cnt_s[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) cnt_s[j] = 0;
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kGroupRows + threadIdx.x;
  if (i < n) atomicAdd(&cnt_s[label[i]], 1);
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) counts[static_cast<int64_t>(blockIdx.x) * k + j] = cnt_s[j];
}

// CTA j: exclusive scan of counts[:, j] over the nblk row blocks (in place), total in
// sizes[j] (one CTA per cluster: the scan is latency-bound, so spread it)
__global__ void __launch_bounds__(1024) group_scan_kernel(int64_t* counts, int64_t nblk, int k,
                                                          int64_t* sizes) {
  __shared__ int64_t wsum[32];
  const int j = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nblk; b0 += blockDim.x) {
    const int64_t b = b0 + threadIdx.x;
    const int64_t v = b < nblk ? counts[b * k + j] : 0;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += t;
      }
      if (lane < nw) wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    incl += warp > 0 ? wsum[warp - 1] : 0;
    if (b < nblk) counts[b * k + j] = carry + incl - v;
    carry += wsum[nw - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) sizes[j] = carry;
}

// start[j] = sum of sizes[0..j) (k is the cluster count: a short serial scan)
__global__ void group_start_kernel(const int64_t* __restrict__ sizes, int k, int64_t* start) {
  if (threadIdx.x != 0) return;
  int64_t run = 0;
  for (int j = 0; j < k; ++j) {
    start[j] = run;
    run += sizes[j];
  }
}

__global__ void group_scatter_kernel(const int32_t* __restrict__ label, int64_t n, int k,
                                     const int64_t* __restrict__ offs,
                                     const int64_t* __restrict__ start, int64_t* members) {
  extern __shared__ int wc[];  // [8][k]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < 8 * k; e += blockDim.x) wc[e] = 0;
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kGroupRows + threadIdx.x;
  const bool valid = i < n;
  const int lab = valid ? label[i] : -1 - lane;  // unique dummies never match real labels
  const unsigned mask = __match_any_sync(0xffffffffu, lab);
  const int rank = __popc(mask & ((1u << lane) - 1u));
  if (valid && rank == 0) wc[warp * k + lab] = __popc(mask);
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    int run = 0;
    for (int w = 0; w < 8; ++w) {
      const int v = wc[w * k + j];
      wc[w * k + j] = run;
      run += v;
    }
  }
  __syncthreads();
  if (valid)
    members[start[lab] + offs[static_cast<int64_t>(blockIdx.x) * k + lab] + wc[warp * k + lab] + rank] = i;
}

void launch_group(const int32_t* label, int64_t n, int k, int64_t* sizes, int64_t* start,
                  int64_t* members, int64_t* tmp, cudaStream_t s, Counter& c) {
  if (n <= 0) return;
  const int64_t nblk = (n + kGroupRows - 1) / kGroupRows;
  group_count_kernel<<<static_cast<unsigned>(nblk), kGroupRows, sizeof(int) * k, s>>>(label, n, k, tmp);
  group_scan_kernel<<<static_cast<unsigned>(k), 1024, 0, s>>>(tmp, nblk, k, sizes);
  group_start_kernel<<<1, 32, 0, s>>>(sizes, k, start);
  group_scatter_kernel<<<static_cast<unsigned>(nblk), kGroupRows, sizeof(int) * 8 * k, s>>>(
      label, n, k, tmp, start, members);
  c.launched(4);
}

// clustering.cpp:34-49: zero, row-order sums, then * (1.0 / size).
// One CTA per (cluster, 32-feature block).  The cluster's member rows (row
// order) stream through a double-buffered shared-memory ring via cp.async; warp
// 0 keeps one strictly sequential accumulator per feature, so every centre
// coordinate is the same chain of roundings as the reference's loop.
#ifndef PKRR_MEANS_F
#define PKRR_MEANS_F 8
#endif
// kMeansF features per CTA: one chain per feature on the consumer warp.  Fewer features
// per CTA = fewer gathered bytes per member row feeding each chain warp and more CTAs:
// C1 per Lloyd iteration 157 us (32) -> 134 (16) -> 120 (8); 4 / 2 exceed one wave (190)
constexpr int kMeansRows = 128, kMeansF = PKRR_MEANS_F, kMeansThreads = 256, kMeansRing = 6;
constexpr int kMeansSmem = kMeansRing * kMeansRows * kMeansF * 8;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Producer/consumer: warps 1-7 stream the member-row chunks into a kMeansRing-deep
// shared ring with cp.async (each loader thread signals the slot's "full"
// mbarrier when its copies land, cp.async.mbarrier.arrive.noinc); warp 0 only runs
// the sequential per-coordinate chains and frees slots through "empty" mbarriers.
// The loaders run up to kMeansRing chunks ahead, so the DADD chain sets the pace.
constexpr int kMeansLoaders = kMeansThreads - 32;

__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(kMeansThreads) means_kernel(const double* __restrict__ X, int64_t d,
                                                              const int64_t* __restrict__ members,
                                                              const int64_t* __restrict__ start,
                                                              const int64_t* __restrict__ sizes, int k,
                                                              double* centers, int bulk, int j0) {
  extern __shared__ double mbuf[];  // [ring][rows][F]
  __shared__ uint64_t full[kMeansRing], empty[kMeansRing];
  const int j = j0 + static_cast<int>(blockIdx.x);
  const int64_t f0 = static_cast<int64_t>(blockIdx.y) * kMeansF;
  const int fw = static_cast<int>(d - f0 < kMeansF ? d - f0 : kMeansF);
  const int64_t sz = sizes[j], st = start[j];
  const int64_t nchunks = (sz + kMeansRows - 1) / kMeansRows;
  if (threadIdx.x == 0) {
    for (int r = 0; r < kMeansRing; ++r) {
      mbar_init(&full[r], kMeansLoaders);
      mbar_init(&empty[r], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (bulk && threadIdx.x >= 32) {
    // Even d, 16-byte aligned X: each member row's feature block is a run of 16-byte
    // pieces.  A loader warp covers kRpw rows per step (kMeansF / 2 lanes per row, one
    // piece per lane); the row indices of chunk c + 1 are loaded while chunk c is
    // issued, so their latency is off the critical path.
    constexpr int kPieces = kMeansF / 2, kRpw = 32 / kPieces, kRps = 7 * kRpw;
    const int w = (threadIdx.x >> 5) - 1, lane = threadIdx.x & 31;
    const int half = lane / kPieces, piece = lane % kPieces;
    const int npieces = fw >> 1;
    constexpr int kSteps = (kMeansRows + kRps - 1) / kRps;
    auto load_idx = [&](int64_t c, int64_t (&ix)[kSteps]) {
#pragma unroll
      for (int u = 0; u < kSteps; ++u) {
        const int rr = kRpw * w + half + kRps * u;
        const int64_t r = c * kMeansRows + rr;
        ix[u] = (c < nchunks && rr < kMeansRows && r < sz) ? __ldg(members + st + r) : -1;
      }
    };
    int64_t cur[kSteps], nxt[kSteps];
    load_idx(0, cur);
    for (int64_t c = 0; c < nchunks; ++c) {
      load_idx(c + 1, nxt);
      const int slot = static_cast<int>(c % kMeansRing);
      mbar_wait(&empty[slot], static_cast<uint32_t>(((c / kMeansRing) & 1) ^ 1));
      double* b = mbuf + slot * kMeansRows * kMeansF;
      if (piece < npieces) {
#pragma unroll
        for (int u = 0; u < kSteps; ++u) {
          const int rr = kRpw * w + half + kRps * u;
          if (cur[u] >= 0)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(b + rr * kMeansF + 2 * piece)),
                         "l"(X + cur[u] * d + f0 + 2 * piece)
                         : "memory");
        }
      }
      cp_async_mbar_arrive_noinc(&full[slot]);
#pragma unroll
      for (int u = 0; u < kSteps; ++u) cur[u] = nxt[u];
    }
    return;
  }
  if (threadIdx.x >= 32) {
    const int l = threadIdx.x - 32;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int slot = static_cast<int>(c % kMeansRing);
      mbar_wait(&empty[slot], static_cast<uint32_t>(((c / kMeansRing) & 1) ^ 1));
      const int64_t r0 = c * kMeansRows;
      const int rows = static_cast<int>(sz - r0 < kMeansRows ? sz - r0 : kMeansRows);
      double* b = mbuf + slot * kMeansRows * kMeansF;
      constexpr int kPer = (kMeansRows * kMeansF + kMeansLoaders - 1) / kMeansLoaders;
      int64_t idx[kPer];
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int e = l + kMeansLoaders * q, r = e / kMeansF;
        idx[q] = (e < kMeansRows * kMeansF && r < rows) ? __ldg(members + st + r0 + r) : -1;
      }
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int e = l + kMeansLoaders * q, r = e / kMeansF, f = e % kMeansF;
        if (idx[q] >= 0 && f < fw) cp_async8(b + r * kMeansF + f, X + idx[q] * d + f0 + f);
      }
      cp_async_mbar_arrive_noinc(&full[slot]);
    }
    return;
  }
  // Consumer: one strictly sequential DADD chain per coordinate (lane).  Full chunks
  // run through a two-buffer register pipeline of 32-row blocks: the next block's 32
  // LDS are in flight while the current block's 32 DADDs run, so the chain advances at
  // the DADD latency.  A slot is released after the DADDs that consumed its last block
  // (their operands -- the LDS results -- have arrived, so the reads are complete).
  double s = 0.0;
  const int64_t nfull = sz / kMeansRows;
  // lanes >= kMeansF run a duplicate chain (never stored) inside the slot
  auto slot_of = [&](int64_t c) {
    return smem_u32(mbuf + (c % kMeansRing) * kMeansRows * kMeansF + (threadIdx.x % kMeansF));
  };
  auto wait_full = [&](int64_t c) {
    mbar_wait(&full[c % kMeansRing], static_cast<uint32_t>((c / kMeansRing) & 1));
  };
  if (nfull > 0) {
    double A[32], B[32];
    wait_full(0);
    {
      const uint32_t b0 = slot_of(0);
#pragma unroll
      for (int u = 0; u < 32; ++u) A[u] = lds_f64_at(b0 + (u * kMeansF) * 8);
    }
    static_assert(kMeansRows == 128, "the block pipeline below assumes 4 blocks of 32 rows per chunk");
    for (int64_t c = 0; c < nfull; ++c) {
      const uint32_t b = slot_of(c);
#pragma unroll
      for (int u = 0; u < 32; ++u) B[u] = lds_f64_at(b + ((32 + u) * kMeansF) * 8);
#pragma unroll
      for (int u = 0; u < 32; ++u) s = __dadd_rn(s, A[u]);
#pragma unroll
      for (int u = 0; u < 32; ++u) A[u] = lds_f64_at(b + ((64 + u) * kMeansF) * 8);
#pragma unroll
      for (int u = 0; u < 32; ++u) s = __dadd_rn(s, B[u]);
#pragma unroll
      for (int u = 0; u < 32; ++u) B[u] = lds_f64_at(b + ((96 + u) * kMeansF) * 8);
      // probe the next chunk's barrier now and branch on it only after this block's
      // DADDs, so the probe latency overlaps the chain
      const uint32_t ready = c + 1 < nfull ? mbar_test(&full[(c + 1) % kMeansRing],
                                                       static_cast<uint32_t>(((c + 1) / kMeansRing) & 1))
                                           : 1u;
#pragma unroll
      for (int u = 0; u < 32; ++u) s = __dadd_rn(s, A[u]);
      if (c + 1 < nfull) {
        if (!ready) wait_full(c + 1);
        const uint32_t bn = slot_of(c + 1);
#pragma unroll
        for (int u = 0; u < 32; ++u) A[u] = lds_f64_at(bn + (u * kMeansF) * 8);
      }
#pragma unroll
      for (int u = 0; u < 32; ++u) s = __dadd_rn(s, B[u]);
      __syncwarp();
      if (threadIdx.x == 0) mbar_arrive(&empty[c % kMeansRing]);
    }
  }
  if (nfull < nchunks) {  // the partial last chunk
    const int64_t c = nfull;
    wait_full(c);
    const uint32_t b = slot_of(c);
    const int rows = static_cast<int>(sz - c * kMeansRows);
    for (int r = 0; r < rows; ++r) s = __dadd_rn(s, lds_f64_at(b + (r * kMeansF) * 8));
  }
  if (threadIdx.x < fw)
    centers[static_cast<int64_t>(j) * d + f0 + threadIdx.x] =
        sz > 0 ? __dmul_rn(s, __ddiv_rn(1.0, static_cast<double>(sz))) : 0.0;
}

void launch_means(const double* X, int64_t d, const int64_t* members, const int64_t* start,
                  const int64_t* sizes, int k, double* centers, cudaStream_t s, Counter& c, int j0, int j1) {
  if (j1 < 0) j1 = k;
  if (j1 <= j0) return;
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, means_kernel, kMeansSmem);
  dim3 grid(j1 - j0, static_cast<unsigned>((d + kMeansF - 1) / kMeansF));
  // 16-byte cp.async pieces need 16-byte aligned rows and an even feature count: even d
  const int bulk = (d % 2 == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0);
  means_kernel<<<grid, kMeansThreads, kMeansSmem, s>>>(X, d, members, start, sizes, k, centers, bulk, j0);
  c.launched();
}

__global__ void label_diff_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n,
                                  unsigned long long* count) {
  unsigned local = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    local += a[i] != b[i];
  if (local) atomicAdd(count, static_cast<unsigned long long>(local));
}

void launch_label_diff(const int32_t* a, const int32_t* b, int64_t n, unsigned long long* count,
                       cudaStream_t s, Counter& c) {
  cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
  label_diff_kernel<<<148 * 2, 256, 0, s>>>(a, b, n, count);
  c.launched();
}

// clustering.cpp:101-110: farthest sample among clusters of size > 1, first index
__global__ void farthest_max_kernel(const double* __restrict__ best, const int32_t* __restrict__ label,
                                    const int64_t* __restrict__ sizes, int64_t n,
                                    unsigned long long* out) {
  unsigned long long m = 0;
  bool any = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = best[i];
    if (sizes[label[i]] <= 1 || !(v >= 0.0)) continue;
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    if (!any || b > m) m = b;
    any = true;
  }
  if (any) atomicMax(&out[0], m + 1);  // +1 so 0 means "no eligible sample"
}

__global__ void farthest_idx_kernel(const double* __restrict__ best, const int32_t* __restrict__ label,
                                    const int64_t* __restrict__ sizes, int64_t n,
                                    unsigned long long* out) {
  const unsigned long long target = out[0];
  if (target == 0) return;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = best[i];
    if (sizes[label[i]] <= 1 || !(v >= 0.0)) continue;
    if (static_cast<unsigned long long>(__double_as_longlong(v)) + 1 == target)
      atomicMin(&out[1], static_cast<unsigned long long>(i));
  }
}

void launch_farthest(const double* best, const int32_t* label, const int64_t* sizes, int64_t n,
                     unsigned long long* out, cudaStream_t s, Counter& c) {
  cudaMemsetAsync(out, 0, sizeof(unsigned long long), s);
  cudaMemsetAsync(out + 1, 0xff, sizeof(unsigned long long), s);
  farthest_max_kernel<<<148 * 4, 256, 0, s>>>(best, label, sizes, n, out);
  farthest_idx_kernel<<<148 * 4, 256, 0, s>>>(best, label, sizes, n, out);
  c.launched(2);
}

__global__ void hist_kernel(const int32_t* __restrict__ label, int64_t row0, int64_t row1, int k,
                            unsigned long long* hist) {
  extern __shared__ int hs[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) hs[j] = 0;
  __syncthreads();
  for (int64_t i = row0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= row1;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int l = label[i];
    if (l >= 0 && l < k) atomicAdd(&hs[l], 1);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    if (hs[j]) atomicAdd(&hist[j], static_cast<unsigned long long>(hs[j]));
}

void launch_hist(const int32_t* label, int64_t row0, int64_t row1, int k, int64_t* hist,
                 cudaStream_t s, Counter& c) {
  cudaMemsetAsync(hist, 0, sizeof(int64_t) * k, s);
  if (row1 < row0) return;
  int64_t blocks = (row1 - row0 + 256) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  hist_kernel<<<static_cast<unsigned>(blocks), 256, sizeof(int) * k, s>>>(
      label, row0, row1, k, reinterpret_cast<unsigned long long*>(hist));
  c.launched();
}

// one CTA per cluster: position of the thr[j]-th occurrence of j in label[row0, n)
__global__ void __launch_bounds__(1024) events_kernel(const int32_t* __restrict__ label, int64_t row0,
                                                      int64_t n, const int64_t* __restrict__ thr,
                                                      int64_t* pos) {
  __shared__ int wsum[32];
  __shared__ int64_t found;
  const int j = blockIdx.x;
  const int64_t need = thr[j];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) found = INT64_MAX;
  __syncthreads();
  if (need <= 0) {
    if (threadIdx.x == 0) pos[j] = INT64_MAX;
    return;
  }
  int64_t run = 0;
  for (int64_t base = row0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool hit = i < n && label[i] == j;
    const unsigned bal = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      if (w < warp) before += wsum[w];
      total += wsum[w];
    }
    const int rank = before + __popc(bal & ((1u << lane) - 1u));
    if (run + total >= need) {
      if (hit && run + rank + 1 == need) found = i;
      __syncthreads();
      break;
    }
    run += total;
    __syncthreads();
  }
  __syncthreads();
  if (threadIdx.x == 0) pos[j] = found;
}

void launch_events(const int32_t* label, int64_t row0, int64_t n, int k, const int64_t* thr,
                   int64_t* pos, cudaStream_t s, Counter& c) {
  events_kernel<<<k, 1024, 0, s>>>(label, row0, n, thr, pos);
  c.launched();
}

// ---------------------------------------------------------------------------
// FP64 tensor-core peak probe
// ---------------------------------------------------------------------------
__global__ void dmma_probe_kernel(double* sink, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) sink[threadIdx.x] = s;
}

void launch_dmma_probe(int blocks, int threads, int iters, double* sink, cudaStream_t s, Counter& c) {
  dmma_probe_kernel<<<blocks, threads, 0, s>>>(sink, iters);
  c.launched();
}

}  // namespace pk

namespace pk {

// ---------------------------------------------------------------------------
// data preparation: standardize (dataset.cpp:178-232) and
// the pairwise distances of auto_sigma_grid (strategies.cpp:204-234), bit-exact
// ---------------------------------------------------------------------------
static bool make_tmap_rows(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld,
                           int box_cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 8)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Column sums and sums of squares in row order (dataset.cpp:211-217): one CTA per 32
// columns; lane j of warp 0 keeps the two strictly sequential chains of column
// f0 + j; a single producer thread streams 64-row x 32-column boxes through a TMA
// ring.  The chains are the rounding sequence of the reference loop, so mean and
// stddev are bitwise the reference's.
constexpr int kStatRows = 64, kStatCols = 32, kStatStages = 8;
constexpr int kStatStageBytes = kStatRows * kStatCols * 8;
constexpr int kStatSmem = kStatStages * kStatStageBytes + 1024 + 256;

__global__ void __launch_bounds__(64) colstats_kernel(const __grid_constant__ CUtensorMap tmX, int64_t n,
                                                      int64_t d, double* __restrict__ mean,
                                                      double* __restrict__ stddev) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStatStages * kStatStageBytes);
  uint64_t* empty = full + kStatStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f0 = blockIdx.x * kStatCols;
  const int64_t nchunks = (n + kStatRows - 1) / kStatRows;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStatStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 1) {
    if (lane == 0) {
      prefetch_tmap(&tmX);
      for (int64_t c = 0; c < nchunks; ++c) {
        const int s = static_cast<int>(c % kStatStages);
        mbar_wait(&empty[s], static_cast<uint32_t>(((c / kStatStages) & 1) ^ 1));
        mbar_arrive_expect_tx(&full[s], kStatStageBytes);
        tma_load_2d(smem + s * kStatStageBytes, &tmX, f0, static_cast<int>(c * kStatRows), &full[s]);
      }
      // do not exit before the last loads have landed (their mbarrier lives in this CTA)
      for (int64_t c = nchunks > kStatStages ? nchunks - kStatStages : 0; c < nchunks; ++c)
        mbar_wait(&full[c % kStatStages], static_cast<uint32_t>((c / kStatStages) & 1));
    }
    return;
  }
  double sum = 0.0, sq = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int s = static_cast<int>(c % kStatStages);
    mbar_wait(&full[s], static_cast<uint32_t>((c / kStatStages) & 1));
    if (c > 0) {  // deferred release of the previous stage (see dgemm_tn_kernel)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[(c - 1) % kStatStages]);
    }
    const uint32_t b = smem_u32(smem + s * kStatStageBytes) + lane * 8;
    const int rows = static_cast<int>(n - c * kStatRows < kStatRows ? n - c * kStatRows : kStatRows);
    int r = 0;
    for (; r + 8 <= rows; r += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = lds_f64_at(b + (r + u) * kStatCols * 8);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sum = __dadd_rn(sum, v[u]);
        sq = __dadd_rn(sq, __dmul_rn(v[u], v[u]));
      }
    }
    for (; r < rows; ++r) {
      const double v = lds_f64_at(b + r * kStatCols * 8);
      sum = __dadd_rn(sum, v);
      sq = __dadd_rn(sq, __dmul_rn(v, v));
    }
  }
  if (f0 + lane < d) {
    // dataset.cpp:218-224
    const double inv_n = __ddiv_rn(1.0, static_cast<double>(n));
    const double mu = __dmul_rn(sum, inv_n);
    double var = __dsub_rn(__dmul_rn(sq, inv_n), __dmul_rn(mu, mu));
    if (var < 0.0) var = 0.0;
    mean[f0 + lane] = mu;
    stddev[f0 + lane] = __dsqrt_rn(var);
  }
}

// apply_feature_stats (dataset.cpp:187-194): (x - mean) / stddev, 0 where stddev == 0
__global__ void standardize_apply_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                         const double* __restrict__ mean, const double* __restrict__ stddev,
                                         double* __restrict__ out) {
  const int64_t total = n * d;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e % d;
    const double sd = stddev[j];
    out[e] = sd == 0.0 ? 0.0 : __ddiv_rn(__dsub_rn(X[e], mean[j]), sd);
  }
}

bool launch_standardize_stats(const double* X, int64_t n, int64_t d, int64_t ld, double* mean, double* stddev,
                              cudaStream_t s, Counter& c) {
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, colstats_kernel, kStatSmem);
  CUtensorMap tm;  // needs a 16-byte aligned base and row pitch (ld even)
  if (!make_tmap_rows(&tm, X, n, d, ld, kStatCols, kStatRows)) return false;
  colstats_kernel<<<static_cast<unsigned>((d + kStatCols - 1) / kStatCols), 64, kStatSmem, s>>>(tm, n, d, mean,
                                                                                              stddev);
  c.launched();
  return true;
}

void launch_standardize_apply(const double* X, int64_t n, int64_t d, const double* mean, const double* stddev,
                              double* out, cudaStream_t s, Counter& c) {
  if (n <= 0) return;
  const int64_t total = n * d;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
  standardize_apply_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(X, n, d, mean, stddev, out);
  c.launched();
}

// auto_sigma_grid distances (strategies.cpp:214-222): pair (i, j), i < j, at the
// reference's push index; sequential dot, (n_i + n_j) - 2 dot, clamp, sqrt
__global__ void pair_dist_kernel(const double* __restrict__ G, const double* __restrict__ norms, int64_t cnt,
                                 int64_t d, double* __restrict__ out) {
  const int64_t total = cnt * (cnt - 1) / 2;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // invert e = i*cnt - i(i+1)/2 + (j - i - 1)
    int64_t i = static_cast<int64_t>((2.0 * cnt - 1.0 - sqrt((2.0 * cnt - 1.0) * (2.0 * cnt - 1.0) - 8.0 * e)) * 0.5);
    auto start = [&](int64_t r) { return r * cnt - r * (r + 1) / 2; };
    while (i > 0 && start(i) > e) --i;
    while (start(i + 1) <= e) ++i;
    const int64_t j = e - start(i) + i + 1;
    const double* a = G + i * d;
    const double* b = G + j * d;
    double dot = 0.0;
    for (int64_t k = 0; k < d; ++k) dot = __dadd_rn(dot, __dmul_rn(a[k], b[k]));
    double d2 = __dsub_rn(__dadd_rn(norms[i], norms[j]), __dmul_rn(2.0, dot));
    if (d2 < 0.0) d2 = 0.0;
    out[e] = __dsqrt_rn(d2);
  }
}

void launch_pair_dist(const double* G, const double* norms, int64_t cnt, int64_t d, double* out, cudaStream_t s,
                      Counter& c) {
  const int64_t total = cnt * (cnt - 1) / 2;
  if (total <= 0) return;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 8);
  pair_dist_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(G, norms, cnt, d, out);
  c.launched();
}

// ---------------------------------------------------------------------------
// building blocks of the distributed (DKRR) factorization, csrc/dist.cu: the same
// kernels as launch_potrf, addressed through explicit row / column origins so that a
// device can work on its own compact column slabs (row-major, ld = its slab width).
// ---------------------------------------------------------------------------
void launch_gemm_update(const CUtensorMap& tmA, const CUtensorMap& tmB, int a_row0, int a_k0, int b_row0, int b_k0,
                        int ktiles, double* C, int64_t ldc, int c_row0, int c_col0, int tiles_m128, int tiles_n,
                        const int* abort, cudaStream_t s, Counter& c) {
  if (tiles_m128 <= 0 || tiles_n <= 0 || ktiles <= 0) return;
  GemmParams u{};
  u.a_row0 = a_row0;
  u.b_row0 = b_row0;
  u.a_k0 = a_k0;
  u.b_k0 = b_k0;
  u.ktiles = ktiles;
  u.C = C;
  u.ldc = ldc;
  u.c_row0 = c_row0;
  u.c_col0 = c_col0;
  u.tiles_n = tiles_n;
  u.abort_flag = abort;
  if (tiles_m128 * tiles_n < g_sms) {  // under one wave of 128-row tiles: 64-row tiles
    u.tiles_m = 2 * tiles_m128;
    gemm_launch<64, G_UPDATE>(tmA, tmB, u, u.tiles_m * tiles_n, s, c);
  } else {
    u.tiles_m = tiles_m128;
    gemm_launch<128, G_UPDATE>(tmA, tmB, u, u.tiles_m * tiles_n, s, c);
  }
}

void launch_gemm_trsm(const CUtensorMap& tmA, const CUtensorMap& tmLinv, int row0, int col0, int kb, int rows128,
                      double* C, int64_t ldc, const double* fz, double* fw, const int* abort, cudaStream_t s,
                      Counter& c) {
  if (rows128 <= 0) return;
  GemmParams t{};
  t.a_row0 = row0;
  t.a_k0 = col0;
  t.b_row0 = kb * kNB;
  t.b_k0 = 0;
  t.ktiles = kNB / kBK;
  t.C = C;
  t.ldc = ldc;
  t.c_row0 = row0;
  t.c_col0 = col0;
  t.tiles_n = 1;
  t.tiles_m = rows128 * 2;
  t.abort_flag = abort;
  t.fz = fz;
  t.fw = fw;
  gemm_launch<64, G_STORE>(tmA, tmLinv, t, t.tiles_m, s, c);
}

void launch_leaf_at(double* A_shifted, int64_t lda, int kb, double* Linv, int* status, int64_t m_valid,
                    const double* w, double* z, cudaStream_t s, Counter& c) {
  static std::atomic<uint64_t> attr{0};
  smem_optin(attr, potrf_leaf_kernel, kLeafSmem);
  launch_pdl(potrf_leaf_kernel, 1, kLeafThreads, kLeafSmem, s, A_shifted, lda, kb, Linv, status, m_valid, 1, w, z);
  c.launched();
}

// Gaussian kernel block K[row0 : row0 + rows, col0 : col0 + cols] (global indices,
// rows % 64 == 0, cols % 128 == 0) written at Cblk (ld ldc); padding rows / columns
// (>= m_valid) are 0 -- the caller sets the diagonal
void launch_gram_block(const CUtensorMap& tmX, const double* norms, int64_t dp, int row0, int col0, int rows,
                       int cols, int64_t m_valid, double sigma, double* Cblk, int64_t ldc, cudaStream_t s,
                       Counter& c) {
  if (rows <= 0 || cols <= 0) return;
  GemmParams p{};
  p.ktiles = static_cast<int>(dp / kBK);
  p.a_row0 = row0;
  p.b_row0 = col0;
  p.C = Cblk;
  p.ldc = ldc;
  p.tiles_m = rows / 64;
  p.tiles_n = cols / 128;
  p.norm_a = norms + row0;
  p.norm_b = norms + col0;
  p.valid_a = static_cast<int>(m_valid - row0 < 0 ? 0 : m_valid - row0);
  p.valid_b = static_cast<int>(m_valid - col0 < 0 ? 0 : m_valid - col0);
  p.denom = (2.0 * sigma) * sigma;
  p.neg_inv_denom = -1.0 / p.denom;
  gemm_launch<64, G_GRAM_CROSS>(tmX, tmX, p, p.tiles_m * p.tiles_n, s, c);
}

__global__ void set_diag_ld_kernel(double* A, int64_t ld, int64_t row0, int64_t col0, int64_t count, double v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < count) A[(row0 + i) * ld + col0 + i] = v;
}

void launch_set_diag(double* A, int64_t ld, int64_t row0, int64_t col0, int64_t count, double v, cudaStream_t s,
                     Counter& c) {
  if (count <= 0) return;
  set_diag_ld_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(A, ld, row0, col0, count, v);
  c.launched();
}

__global__ void fill_flags_kernel(int* f, int n, int lo, int hi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = i >= lo && i < hi ? 0 : 1;
}

void launch_trsv_bwd_range(const double* L_shifted, int64_t ld, const double* Linv, const double* z, double* x, int nb,
                           int ilo, int ihi, int* scratch, const int* abort, cudaStream_t s, Counter& c) {
  // scratch: [0] ticket, [1 ..] flags: the blocks >= ihi are final (x from later super-columns)
  cudaMemsetAsync(scratch, 0, sizeof(int), s);
  fill_flags_kernel<<<(nb + 255) / 256, 256, 0, s>>>(scratch + 1, nb, ilo, ihi);
  trsv_bwd_optin();
  trsv_bwd_kernel<<<ihi - ilo, 256, kTrsvBwdSmem, s>>>(L_shifted, ld, Linv, z, x, nb, scratch, scratch + 1, abort, ihi,
                                                       nullptr);
  c.launched(2);
}

}  // namespace pk
