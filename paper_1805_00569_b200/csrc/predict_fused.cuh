// predict_fused.cuh -- prediction with the test-by-support kernel tile fused into the
// alpha contraction (strategies.cpp:284-294 builds K(test, part) and multiplies by
// alpha; kernel.cpp:52-56 is the Gaussian):
//
//   pred[q] = sum_i exp(-max(0, (n_q + n_i) - 2 x_q.x_i) / ((2 s) s)) * alpha[i]
//
// No cross matrix is materialised.  A CTA owns 64 query rows x a chunk of support
// tiles (128 rows each): per tile it runs the same TMA + DMMA dot-product mainloop as
// the gram (gemm_dmma.cuh: 4-stage 128B-swizzled ring, warp 8 produces, warps 0-7
// multiply on a 2 x 4 grid), applies the Gaussian in registers and folds the tile into
// per-row partial sums against alpha.  The producer runs ahead across tile boundaries,
// so the epilogue of tile t overlaps the loads of tile t+1.  Per-(chunk, row) partials
// land in a scratch array; predict_reduce_kernel adds the chunks in a fixed order, so
// the prediction is deterministic.
#pragma once

#include "gemm_dmma.cuh"

namespace pk {

struct PredictParams {
  int ktiles;             // dp / 16
  int tiles_q, tiles_x;   // qp / 64, mp / 128
  int chunk;              // support tiles per CTA
  int valid_x;            // support rows >= valid_x are padding (contribute 0)
  int64_t qp;
  const double* qnorms;
  const double* xnorms;
  const double* alpha;
  double neg_inv_denom;   // -1 / ((2 s) s)
  double* partial;        // [nchunks][qp]
  const int* abort_flag;  // per-part NPD flag: nothing to predict with
};

__global__ void __launch_bounds__(kGemmThreads, 1)
    predict_fused_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX,
                         PredictParams p) {
  using Cfg = GemmCfg<64>;
  if (p.abort_flag && *reinterpret_cast<const volatile int*>(p.abort_flag)) return;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::STAGE_BYTES);
  uint64_t* empty = full + kStages;
  __shared__ double red[4][64];

  const int tq = blockIdx.x % p.tiles_q, ch = blockIdx.x / p.tiles_q;
  const int t0 = ch * p.chunk, t1 = min(p.tiles_x, t0 + p.chunk);
  const int KT = p.ktiles, total = (t1 - t0) * KT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    if (lane == 0) {
      prefetch_tmap(&tmQ);
      prefetch_tmap(&tmX);
      for (int g = 0; g < total; ++g) {
        const int tn = t0 + g / KT, kt = g % KT;
        const int s = g % kStages;
        const uint32_t ph = (g / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        unsigned char* sa = smem + s * Cfg::STAGE_BYTES;
        unsigned char* sb = sa + Cfg::A_BYTES;
        tma_load_2d(sa, &tmQ, kt * kBK, tq * 64, &full[s]);
        tma_load_2d(sb, &tmX, kt * kBK, tn * kBN, &full[s]);
        tma_load_2d(sb + 8192, &tmX, kt * kBK, tn * kBN + 64, &full[s]);
      }
    }
    return;
  }

  const int wm = warp >> 2, wn = warp & 3;
  const int lr = lane >> 2, lk = lane & 3;
  double na[Cfg::MT], part[Cfg::MT];
#pragma unroll
  for (int i = 0; i < Cfg::MT; ++i) {
    na[i] = __ldg(p.qnorms + tq * 64 + wm * Cfg::WM + lr + i * 8);
    part[i] = 0.0;
  }
  int g = 0;
  for (int tn = t0; tn < t1; ++tn) {
    // this tile's support norms and alpha, loaded before its mainloop
    const int gj0 = tn * kBN + wn * Cfg::WN + 2 * lk;
    double nb[Cfg::NT][2], al[Cfg::NT][2];
#pragma unroll
    for (int j = 0; j < Cfg::NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        nb[j][e] = __ldg(p.xnorms + gj0 + j * 8 + e);
        al[j][e] = __ldg(p.alpha + gj0 + j * 8 + e);
      }
    double acc[Cfg::MT][Cfg::NT][2];
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < KT; ++kt, ++g) {
      const int s = g % kStages;
      mbar_wait(&full[s], (g / kStages) & 1);
      if (g > 0) {  // deferred release (see gemm_dmma.cuh)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[(g - 1) % kStages]);
      }
      const unsigned char* sa = smem + s * Cfg::STAGE_BYTES;
      const unsigned char* sb = sa + Cfg::A_BYTES;
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        const int k = ks * 4 + lk;
        double af[Cfg::MT], bf[Cfg::NT];
#pragma unroll
        for (int i = 0; i < Cfg::MT; ++i) af[i] = lds_f64(sa, swz128(wm * Cfg::WM + i * 8 + lr, k));
#pragma unroll
        for (int j = 0; j < Cfg::NT; ++j) bf[j] = lds_f64(sb, swz128(wn * Cfg::WN + j * 8 + lr, k));
#pragma unroll
        for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::NT; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
    }
    // Gaussian (kernel.cpp:52-56, same arithmetic as the gram epilogue) x alpha
#pragma unroll
    for (int j = 0; j < Cfg::NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (gj0 + j * 8 + e >= p.valid_x) continue;
        double ex[Cfg::MT];  // the column's MT exp chains, interleaved stage by stage
#pragma unroll
        for (int i = 0; i < Cfg::MT; ++i) {
          double dist2 = (na[i] + nb[j][e]) - 2.0 * acc[i][j][e];
          dist2 = dist2 < 0.0 ? 0.0 : dist2;
          ex[i] = dist2 * p.neg_inv_denom;
        }
        exp_nonpos_n<Cfg::MT>(ex);
#pragma unroll
        for (int i = 0; i < Cfg::MT; ++i) part[i] = fma(ex[i], al[j][e], part[i]);
      }
  }
  // rows: 4 lanes (lk) x 4 warps (wn) hold partials of the same row; fixed-order sums
#pragma unroll
  for (int i = 0; i < Cfg::MT; ++i) {
    part[i] += __shfl_xor_sync(0xffffffffu, part[i], 1);
    part[i] += __shfl_xor_sync(0xffffffffu, part[i], 2);
    if (lk == 0) red[wn][wm * Cfg::WM + lr + i * 8] = part[i];
  }
  consumer_sync(kConsumerWarps * 32);
  if (threadIdx.x < 64) {
    const int r = threadIdx.x;
    p.partial[ch * p.qp + tq * 64 + r] = ((red[0][r] + red[1][r]) + red[2][r]) + red[3][r];
  }
}

__global__ void __launch_bounds__(256) predict_reduce_kernel(const double* __restrict__ partial, int64_t qp,
                                                             int nchunks, int64_t count,
                                                             double* __restrict__ pred, const int* abort) {
  if (abort && *reinterpret_cast<const volatile int*>(abort)) return;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= count) return;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += partial[c * qp + r];
  pred[r] = s;
}

}  // namespace pk
