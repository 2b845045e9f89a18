// dist.cu -- DKRR: ONE Gaussian KRR system factorised across the GPUs of a group
// (pkrrgpu_multi).  The paper's whole-data baseline (distributed kernel
// creation + a ScaLAPACK Cholesky; the reference keeps it as a cost formula only,
// runtime.cpp:54-57), and the way past one GPU's HBM for an exact solve.
//
// Layout: the padded system (mp = m rounded up to the super-column width Ws = 128 G) is
// cut into nbs = mp / Ws super-columns; super-column c belongs to device c mod W and is
// stored there COMPACTLY, row-major [mp x nloc Ws] (slot j = its j-th owned
// super-column; rows < c Ws of a slot are unused).  So each GPU holds ~1/W of the matrix.
//
// Right-looking blocked Cholesky, one super-column per step k (owner o = k mod W):
//   1. o factors super-column k in place: per 128-column panel kb, the column update by
//      the super-column's earlier panels (DMMA GEMM), the leaf (potrf_leaf_kernel: 128 x
//      128 block + its inverse) and the panel TRSM (DMMA GEMM with inv(L_kb)), the
//      forward substitution fused (w -= L21 z_kb), exactly the kernels of launch_potrf;
//   2. every other device copies the factored panel (rows >= k Ws, Ws wide) into its
//      panel buffer -- a peer copy over NVLink / NVSwitch (cudaMemcpy2DAsync on UVA),
//      ordered after o's factorisation by a cross-device event;
//   3. every device subtracts panel k from each of its super-columns c > k
//      (C -= P P^T, K = Ws, one DMMA GEMM per column).  Lookahead: the owner of k + 1
//      updates column k + 1 first, factors it, and only then updates its other columns,
//      so the next panel is ready while the other devices are still updating.
// The forward-substitution vector w and, after the factorisation, the backward solve's
// x travel owner to owner along the super-column chain (backward: trsv_bwd_kernel over
// each super-column's blocks with the later x blocks final).  One host thread enqueues
// everything; devices synchronise only through events, and two contexts may share one
// GPU (this build's test configuration).
//
// Every element of the factor receives the panels' contributions in increasing order;
// only the grouping of the updates differs from the one-GPU schedule (K = Ws per GEMM
// instead of the recursive group blocking), so alpha agrees with pkrrgpu_train_krr to
// rounding (tests: <= 1e-8 relative at the conditioning of the test systems).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/pkrr_gpu.h"
#include "kernels.cuh"

extern "C" void pkrrgpu_set_last_error_(const char* msg);
extern "C" int pkrrgpu_multi_device_(const pkrrgpu_multi* m, int i);
extern "C" void pkrrgpu_add_launches_(pkrrgpu_ctx* ctx, int64_t n);
extern "C" int pkrrgpu_context_device_(const pkrrgpu_ctx* ctx);

namespace {

using pk::kNB;
constexpr int kBK = 16;  // f64 per k-tile of the DMMA GEMM (gemm_dmma.cuh)

struct DistFail {
  int code;
  std::string msg;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DistFail{PKRRGPU_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

struct Dev {
  int dev = 0;
  pkrrgpu_ctx* ctx = nullptr;
  cudaStream_t s = nullptr;
  pk::Counter cnt;
  std::vector<int> cols;  // owned super-columns, slot order
  int64_t ld = 0;         // nloc * Ws
  double* A = nullptr;    // [mp x ld]
  double* Linv = nullptr; // [mp x 128]
  double* P[2] = {nullptr, nullptr};  // panel buffers [mp x Ws] (global rows)
  double *w = nullptr, *z = nullptr, *x = nullptr, *Xp = nullptr, *norms = nullptr, *y = nullptr;
  int* status = nullptr;
  int* scratch = nullptr;
  CUtensorMap tmA, tmLinv, tmP[2], tmX;
  std::vector<void*> allocs;

  template <typename T>
  T* alloc(int64_t count, bool zero = false) {
    void* p = nullptr;
    ck(cudaMalloc(&p, sizeof(T) * static_cast<size_t>(count > 0 ? count : 1)), "cudaMalloc");
    allocs.push_back(p);
    if (zero) ck(cudaMemsetAsync(p, 0, sizeof(T) * static_cast<size_t>(count > 0 ? count : 1), s), "memset");
    return static_cast<T*>(p);
  }
  int slot(int c) const { return static_cast<int>(std::find(cols.begin(), cols.end(), c) - cols.begin()); }
};

struct Geom {
  int W = 1, G = 8;
  int64_t n = 0, d = 0, Ws = 0, mp = 0, nb = 0, nbs = 0, dp = 0;
  double sigma = 1.0, shift = 0.0;
  int owner(int64_t c) const { return static_cast<int>(c % W); }
};

Geom make_geom(int W, int64_t n, int64_t d, double sigma, double lambda) {
  Geom g;
  g.W = W;
  // super-column width: 128 G columns; G = 16 (K = 2048 per update GEMM) for large
  // systems, 8 below 16384 rows, fewer when that leaves a device without a column
  g.G = n >= 16384 ? 16 : 8;
  if (const char* e = std::getenv("PKRR_DIST_GROUP")) g.G = std::max(1, std::atoi(e));
  while (g.G > 1 && (n + 128 * g.G - 1) / (128 * g.G) < W) g.G /= 2;
  g.n = n;
  g.d = d;
  g.Ws = kNB * g.G;
  g.mp = (n + g.Ws - 1) / g.Ws * g.Ws;
  g.nb = g.mp / kNB;
  g.nbs = g.mp / g.Ws;
  g.dp = (d + 15) / 16 * 16;
  g.sigma = sigma;
  g.shift = lambda * static_cast<double>(n);
  return g;
}

// allocations, inputs, and the device's own super-columns of A = K + lambda n I
// (kernel.cpp:81-141; the diagonal exactly 1 + shift).  panel_extra: doubles appended
// to each panel buffer (the one-process-per-GPU variant ships w and a status with it).
void setup_dev(Dev& v, const Geom& g, int r, const double* X, const double* y, bool panels, int64_t panel_extra) {
  const int64_t mp = g.mp, Ws = g.Ws, dp = g.dp;
  ck(cudaSetDevice(v.dev), "cudaSetDevice");
  ck(cudaStreamCreateWithFlags(&v.s, cudaStreamNonBlocking), "stream");
  for (int64_t c = r; c < g.nbs; c += g.W) v.cols.push_back(static_cast<int>(c));
  v.ld = std::max<int64_t>(1, static_cast<int64_t>(v.cols.size())) * Ws;
  v.A = v.alloc<double>(mp * v.ld);
  v.Linv = v.alloc<double>(mp * kNB, true);  // the leaf writes only the lower 32-blocks
  if (panels) {
    v.P[0] = v.alloc<double>(mp * Ws + panel_extra);
    v.P[1] = v.alloc<double>(mp * Ws + panel_extra);
  }
  v.w = v.alloc<double>(mp, true);
  v.z = v.alloc<double>(mp, true);
  v.x = v.alloc<double>(mp, true);
  v.y = v.alloc<double>(mp, true);
  v.Xp = v.alloc<double>(mp * dp, true);
  v.norms = v.alloc<double>(mp);
  v.status = v.alloc<int>(2, true);
  v.scratch = v.alloc<int>(g.nb + 1, true);
  ck(cudaMemcpy2DAsync(v.Xp, sizeof(double) * dp, X, sizeof(double) * g.d, sizeof(double) * g.d, g.n,
                       cudaMemcpyDefault, v.s),
     "copy X");
  ck(cudaMemcpyAsync(v.y, y, sizeof(double) * g.n, cudaMemcpyDefault, v.s), "copy y");
  if (!pk::make_tmap(&v.tmA, v.A, mp, v.ld, v.ld) || !pk::make_tmap(&v.tmLinv, v.Linv, mp, kNB, kNB) ||
      !pk::make_tmap(&v.tmX, v.Xp, mp, dp, dp))
    throw DistFail{PKRRGPU_CUDA, "tensor map"};
  for (int b = 0; b < 2; ++b)
    if (v.P[b] && !pk::make_tmap(&v.tmP[b], v.P[b], mp, Ws, Ws)) throw DistFail{PKRRGPU_CUDA, "tensor map"};
  pk::launch_row_norms(v.Xp, mp, dp, dp, v.norms, v.s, v.cnt);
  for (size_t j = 0; j < v.cols.size(); ++j) {
    const int64_t c = v.cols[j];
    double* blk = v.A + c * Ws * v.ld + static_cast<int64_t>(j) * Ws;
    pk::launch_gram_block(v.tmX, v.norms, dp, static_cast<int>(c * Ws), static_cast<int>(c * Ws),
                          static_cast<int>(mp - c * Ws), static_cast<int>(Ws), g.n, g.sigma, blk, v.ld, v.s, v.cnt);
    pk::launch_set_diag(v.A, v.ld, c * Ws, static_cast<int64_t>(j) * Ws, Ws, 1.0 + g.shift, v.s, v.cnt);
  }
}

// factor super-column k in place on its owner: per 128-column panel the column update by
// the super-column's earlier panels, the leaf, the panel TRSM (forward substitution fused)
void factor_supercol(Dev& v, const Geom& g, int64_t k) {
  const int64_t j = v.slot(static_cast<int>(k)), Ws = g.Ws, G = g.G;
  double* shifted = v.A + j * Ws - k * Ws;  // block (kb, kb) at shifted + 128 kb (ld + 1)
  for (int64_t kb = k * G; kb < (k + 1) * G; ++kb) {
    const int col = static_cast<int>(j * Ws + (kb - k * G) * kNB);
    if (kb > k * G)
      pk::launch_gemm_update(v.tmA, v.tmA, static_cast<int>(kb * kNB), static_cast<int>(j * Ws),
                             static_cast<int>(kb * kNB), static_cast<int>(j * Ws),
                             static_cast<int>((kb - k * G) * (kNB / kBK)), v.A, v.ld, static_cast<int>(kb * kNB), col,
                             static_cast<int>(g.nb - kb), 1, v.status, v.s, v.cnt);
    pk::launch_leaf_at(shifted, v.ld, static_cast<int>(kb), v.Linv, v.status, g.n, v.w, v.z, v.s, v.cnt);
    pk::launch_gemm_trsm(v.tmA, v.tmLinv, static_cast<int>((kb + 1) * kNB), col, static_cast<int>(kb),
                         static_cast<int>(g.nb - 1 - kb), v.A, v.ld, v.z + kb * kNB, v.w, v.status, v.s, v.cnt);
  }
}

// panel k (source: tensor map src, its K columns starting at k0) applied to super-column c
void apply_panel(Dev& v, const Geom& g, const CUtensorMap& src, int k0, int64_t c) {
  const int64_t Ws = g.Ws;
  pk::launch_gemm_update(src, src, static_cast<int>(c * Ws), k0, static_cast<int>(c * Ws), k0,
                         static_cast<int>(Ws / kBK), v.A, v.ld, static_cast<int>(c * Ws),
                         static_cast<int>(v.slot(static_cast<int>(c)) * Ws), static_cast<int>((g.mp - c * Ws) / kNB),
                         g.G, v.status, v.s, v.cnt);
}

// ||(K + lambda n I) alpha - y|| / ||y|| (solver.cpp:103-119), K alpha recomputed by the
// fused kernel-tile x alpha contraction (no stored K)
double residual_of(Dev& v, const Geom& g) {
  double* partial = v.alloc<double>(pk::predict_partial_elems(g.mp, g.mp));
  double* Ka = v.alloc<double>(g.mp * pk::kSymvSplit, true);
  double* res = v.alloc<double>(2, true);
  pk::launch_predict_fused(v.tmX, v.tmX, v.norms, v.norms, g.mp, g.n, g.mp, g.n, g.dp, g.sigma, v.x, partial, Ka,
                           nullptr, v.s, v.cnt);
  pk::launch_residual_finish(Ka, v.x, v.y, g.n, g.shift, res, nullptr, v.s, v.cnt);
  double h[2];
  ck(cudaMemcpyAsync(h, res, sizeof(h), cudaMemcpyDeviceToHost, v.s), "copy residual");
  ck(cudaStreamSynchronize(v.s), "sync");
  return h[1];
}

}  // namespace

extern "C" int pkrrgpu_multi_train_krr(pkrrgpu_multi* mg, const double* X, const double* y, int64_t n, int64_t d,
                                       double sigma, double lambda, double* alpha, double* residual,
                                       int64_t* npd_pivot) {
  std::vector<Dev> D;
  std::vector<cudaEvent_t> events;
  int rc = PKRRGPU_OK;
  try {
    if (!mg || !X || !y || n <= 0 || d <= 0) throw DistFail{PKRRGPU_INVALID, "train_krr: empty dataset"};
    if (!(lambda > 0.0)) throw DistFail{PKRRGPU_INVALID, "train_krr: lambda must be > 0"};
    if (!(sigma > 0.0)) throw DistFail{PKRRGPU_INVALID, "gaussian kernel needs sigma > 0"};
    const int W = pkrrgpu_multi_size(mg);
    const Geom g = make_geom(W, n, d, sigma, lambda);
    const int64_t Ws = g.Ws, mp = g.mp, nb = g.nb, nbs = g.nbs, G = g.G;
    auto owner = [&](int64_t c) { return g.owner(c); };
    D.resize(W);
    for (int r = 0; r < W; ++r) {
      D[r].dev = pkrrgpu_multi_device_(mg, r);
      D[r].ctx = pkrrgpu_multi_context(mg, r);
      setup_dev(D[r], g, r, X, y, W > 1, 0);
    }
    // forward-substitution accumulator w := y on the first owner
    ck(cudaSetDevice(D[0].dev), "cudaSetDevice");
    ck(cudaMemcpyAsync(D[0].w, D[0].y, sizeof(double) * mp, cudaMemcpyDeviceToDevice, D[0].s), "w");

    auto new_event = [&](Dev& v) {
      cudaEvent_t e;
      ck(cudaSetDevice(v.dev), "cudaSetDevice");
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      ck(cudaEventRecord(e, v.s), "event");
      events.push_back(e);
      return e;
    };
    // panel k applied to super-column c of device v (source: its own slab or its buffer)
    auto apply = [&](Dev& v, int64_t k, int64_t c) {
      const bool own = owner(k) == static_cast<int>(&v - D.data());
      apply_panel(v, g, own ? v.tmA : v.tmP[k & 1], own ? static_cast<int>(v.slot(static_cast<int>(k)) * Ws) : 0, c);
    };
    auto bulk = [&](Dev& v, int64_t k, int64_t skip) {
      for (int c : v.cols)
        if (c > k && c != skip) apply(v, k, c);
    };

    std::vector<cudaEvent_t> ev_fact(nbs, nullptr);
    std::vector<int64_t> pending(W, -1);
    for (int64_t k = 0; k < nbs; ++k) {
      const int o = owner(k);
      Dev& v = D[o];
      ck(cudaSetDevice(v.dev), "cudaSetDevice");
      if (k > 0 && owner(k - 1) != o) {  // the forward-substitution vector from the previous owner
        ck(cudaStreamWaitEvent(v.s, ev_fact[k - 1], 0), "wait");
        ck(cudaMemcpyAsync(v.w + k * Ws, D[owner(k - 1)].w + k * Ws, sizeof(double) * (mp - k * Ws),
                           cudaMemcpyDefault, v.s),
           "copy w");
      }
      // ---- factor super-column k in place ----
      const int64_t j = v.slot(static_cast<int>(k));
      factor_supercol(v, g, k);
      ev_fact[k] = new_event(v);
      if (pending[o] == k - 1 && k > 0) {  // lookahead: the rest of panel k-1 after factoring k
        bulk(v, k - 1, k);
        pending[o] = -1;
      }
      for (int r = 0; r < W; ++r) {
        Dev& u = D[r];
        ck(cudaSetDevice(u.dev), "cudaSetDevice");
        if (r != o) {  // panel k (rows >= k Ws) into this device's buffer
          ck(cudaStreamWaitEvent(u.s, ev_fact[k], 0), "wait");
          ck(cudaMemcpy2DAsync(u.P[k & 1] + k * Ws * Ws, sizeof(double) * Ws, v.A + k * Ws * v.ld + j * Ws,
                               sizeof(double) * v.ld, sizeof(double) * Ws, mp - k * Ws, cudaMemcpyDefault, u.s),
             "copy panel");
        }
        if (k + 1 < nbs && owner(k + 1) == r) {
          apply(u, k, k + 1);  // lookahead column first
          pending[r] = k;
        } else {
          bulk(u, k, -1);
        }
      }
    }
    // ---- backward solve L^T x = z along the chain, last super-column first ----
    std::vector<cudaEvent_t> ev_bwd(nbs, nullptr);
    for (int64_t k = nbs - 1; k >= 0; --k) {
      const int o = owner(k);
      Dev& v = D[o];
      ck(cudaSetDevice(v.dev), "cudaSetDevice");
      if (k < nbs - 1 && owner(k + 1) != o) {
        ck(cudaStreamWaitEvent(v.s, ev_bwd[k + 1], 0), "wait");
        ck(cudaMemcpyAsync(v.x + (k + 1) * Ws, D[owner(k + 1)].x + (k + 1) * Ws,
                           sizeof(double) * (mp - (k + 1) * Ws), cudaMemcpyDefault, v.s),
           "copy x");
      }
      const int64_t j = v.slot(static_cast<int>(k));
      pk::launch_trsv_bwd_range(v.A + j * Ws - k * Ws, v.ld, v.Linv, v.z, v.x, static_cast<int>(nb),
                                static_cast<int>(k * G), static_cast<int>((k + 1) * G), v.scratch, v.status, v.s,
                                v.cnt);
      ev_bwd[k] = new_event(v);
    }
    // ---- status: the first failing pivot over the devices (solver.cpp:19-20) ----
    int64_t piv = -1;
    for (auto& v : D) {
      ck(cudaSetDevice(v.dev), "cudaSetDevice");
      ck(cudaStreamSynchronize(v.s), "dkrr");
      int st[2] = {0, 0};
      ck(cudaMemcpy(st, v.status, sizeof(st), cudaMemcpyDeviceToHost), "status");
      if (st[0] && (piv < 0 || st[1] < piv)) piv = st[1];
      if (v.cnt.err != cudaSuccess)
        throw DistFail{PKRRGPU_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(v.cnt.err)};
    }
    if (piv >= 0) {
      if (npd_pivot) *npd_pivot = piv;
      throw DistFail{PKRRGPU_NPD, "matrix not positive definite: pivot " + std::to_string(piv)};
    }
    Dev& z0 = D[0];  // x complete on the owner of super-column 0
    ck(cudaSetDevice(z0.dev), "cudaSetDevice");
    if (alpha) ck(cudaMemcpy(alpha, z0.x, sizeof(double) * n, cudaMemcpyDefault), "copy alpha");
    if (residual) *residual = residual_of(z0, g);
    for (auto& v : D)
      if (v.cnt.err != cudaSuccess)
        throw DistFail{PKRRGPU_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(v.cnt.err)};
  } catch (const DistFail& f) {
    pkrrgpu_set_last_error_(f.msg.c_str());
    rc = f.code;
  }
  for (auto& v : D) {
    cudaSetDevice(v.dev);
    if (v.s) cudaStreamSynchronize(v.s);
    for (void* p : v.allocs) cudaFree(p);
    if (v.s) cudaStreamDestroy(v.s);
    if (v.ctx) pkrrgpu_add_launches_(v.ctx, v.cnt.launches);
  }
  for (auto e : events) cudaEventDestroy(e);
  return rc;
}

// ---------------------------------------------------------------------------------
// DKRR with one process per GPU: the same algorithm, every rank running its own share
// (super-columns c with c mod world == rank) on its context; the exchange is the
// caller's broadcast (an NCCL broadcast over NVLink in bench / torch.distributed; a
// host-staged one for the gloo tests).  Step k: the owner factors super-column k and
// packs [panel rows >= k Ws | the forward-substitution vector w | its NPD status] into a
// panel buffer; one broadcast from the owner; every rank applies the panel to its
// super-columns > k.  Backward: the owner of k solves its blocks and broadcasts them.
// ---------------------------------------------------------------------------------
extern "C" int pkrrgpu_dist_train_krr(pkrrgpu_ctx* ctx, int rank, int world, pkrrgpu_bcast_fn bcast, void* user,
                                      const double* X, const double* y, int64_t n, int64_t d, double sigma,
                                      double lambda, double* alpha, double* residual, int64_t* npd_pivot) {
  Dev v;
  int rc = PKRRGPU_OK;
  try {
    if (!ctx || !X || !y || n <= 0 || d <= 0) throw DistFail{PKRRGPU_INVALID, "train_krr: empty dataset"};
    if (!(lambda > 0.0)) throw DistFail{PKRRGPU_INVALID, "train_krr: lambda must be > 0"};
    if (!(sigma > 0.0)) throw DistFail{PKRRGPU_INVALID, "gaussian kernel needs sigma > 0"};
    if (world < 1 || rank < 0 || rank >= world || (world > 1 && !bcast))
      throw DistFail{PKRRGPU_INVALID, "dist_train_krr: bad rank / world / broadcast"};
    const Geom g = make_geom(world, n, d, sigma, lambda);
    const int64_t Ws = g.Ws, mp = g.mp, nbs = g.nbs, G = g.G;
    v.ctx = ctx;
    v.dev = pkrrgpu_context_device_(ctx);
    // panel buffer: [mp x Ws panel | mp (w) | 2 (status flag, pivot)]
    const int64_t extra = mp + 2;
    setup_dev(v, g, rank, X, y, true, extra);
    ck(cudaMemcpyAsync(v.w, v.y, sizeof(double) * mp, cudaMemcpyDeviceToDevice, v.s), "w");
    auto exchange = [&](void* buf, int64_t bytes, int root) {
      ck(cudaStreamSynchronize(v.s), "sync");
      if (world > 1 && bcast(user, buf, bytes, root) != 0) throw DistFail{PKRRGPU_CUDA, "DKRR broadcast failed"};
    };
    int64_t piv = -1;
    for (int64_t k = 0; k < nbs; ++k) {
      const int o = g.owner(k);
      double* P = v.P[k & 1];
      double* Pw = P + mp * Ws;
      if (rank == o) {
        factor_supercol(v, g, k);
        const int64_t j = v.slot(static_cast<int>(k));
        ck(cudaMemcpy2DAsync(P + k * Ws * Ws, sizeof(double) * Ws, v.A + k * Ws * v.ld + j * Ws,
                             sizeof(double) * v.ld, sizeof(double) * Ws, mp - k * Ws, cudaMemcpyDeviceToDevice, v.s),
           "pack panel");
        ck(cudaMemcpyAsync(Pw, v.w, sizeof(double) * mp, cudaMemcpyDeviceToDevice, v.s), "pack w");
        int st[2];
        ck(cudaMemcpyAsync(st, v.status, sizeof(st), cudaMemcpyDeviceToHost, v.s), "status");
        ck(cudaStreamSynchronize(v.s), "sync");
        const double flag[2] = {static_cast<double>(st[0]), static_cast<double>(st[1])};
        ck(cudaMemcpyAsync(Pw + mp, flag, sizeof(flag), cudaMemcpyHostToDevice, v.s), "pack status");
      }
      // panel rows k Ws .. mp, then w and the status (contiguous from row k Ws)
      exchange(P + k * Ws * Ws, sizeof(double) * ((mp - k * Ws) * Ws + extra), o);
      if (rank != o) ck(cudaMemcpyAsync(v.w, Pw, sizeof(double) * mp, cudaMemcpyDeviceToDevice, v.s), "w");
      double flag[2];
      ck(cudaMemcpyAsync(flag, Pw + mp, sizeof(flag), cudaMemcpyDeviceToHost, v.s), "status");
      ck(cudaStreamSynchronize(v.s), "sync");
      if (flag[0] != 0.0) {  // NPD on the owner: the first failing column (solver.cpp:19-20)
        piv = static_cast<int64_t>(flag[1]);
        break;
      }
      for (int c : v.cols)
        if (c > k) apply_panel(v, g, v.tmP[k & 1], 0, c);
    }
    if (piv >= 0) {
      if (npd_pivot) *npd_pivot = piv;
      throw DistFail{PKRRGPU_NPD, "matrix not positive definite: pivot " + std::to_string(piv)};
    }
    for (int64_t k = nbs - 1; k >= 0; --k) {
      const int o = g.owner(k);
      if (rank == o) {
        const int64_t j = v.slot(static_cast<int>(k));
        pk::launch_trsv_bwd_range(v.A + j * Ws - k * Ws, v.ld, v.Linv, v.z, v.x, static_cast<int>(g.nb),
                                  static_cast<int>(k * G), static_cast<int>((k + 1) * G), v.scratch, v.status, v.s,
                                  v.cnt);
      }
      exchange(v.x + k * Ws, sizeof(double) * Ws, o);
    }
    ck(cudaStreamSynchronize(v.s), "dkrr");
    if (v.cnt.err != cudaSuccess)
      throw DistFail{PKRRGPU_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(v.cnt.err)};
    if (alpha) ck(cudaMemcpy(alpha, v.x, sizeof(double) * n, cudaMemcpyDefault), "copy alpha");
    if (residual) *residual = residual_of(v, g);
  } catch (const DistFail& f) {
    pkrrgpu_set_last_error_(f.msg.c_str());
    rc = f.code;
  }
  if (v.s) {
    cudaStreamSynchronize(v.s);
    for (void* p : v.allocs) cudaFree(p);
    cudaStreamDestroy(v.s);
  }
  if (ctx) pkrrgpu_add_launches_(ctx, v.cnt.launches);
  return rc;
}
