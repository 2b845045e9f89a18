// gemm_dmma.cuh -- the FP64 tensor-core tile engine behind every O(m^2 d) and
// O(m^3) step of the path:
//
//   G_UPDATE     C -= A B^T        Cholesky trailing update (SYRK on lower tiles)
//   G_STORE      C  = A B^T        panel TRSM as A21 * inv(L11)^T (in place by rows)
//   G_GRAM_SYM   K  = exp(-max(0, n_i + n_j - 2 x_i.x_j) / (2 s^2))   kernel.cpp:52-56,
//                lower tiles computed once and mirrored (kernel.cpp:107-119)
//   G_GRAM_CROSS K(q, i) = same kernel, rectangular (strategies.cpp:284-294)
//
// Operands are row-major "rows x K" f64 matrices read through 2-D TMA tensor maps
// (box 16 x 64, 128B swizzle) into a 4-stage shared-memory ring; warp 8 is the
// TMA producer, warps 0-7 run DMMA (mma.sync m8n8k4 f64) on a 2 x 4 warp grid.
// Accumulators live in registers (tcgen05/TMEM has no FP64 kind on sm_100a).
#pragma once

#include "common.cuh"

namespace pk {

enum GemmMode { G_UPDATE = 0, G_STORE = 1, G_GRAM_SYM = 2, G_GRAM_CROSS = 3 };

struct GemmParams {
  int a_row0, b_row0;  // operand row origins (tile tm reads rows a_row0 + tm*BM ...)
  int a_k0, b_k0;      // operand column origins of the K range
  int ktiles;          // K extent = 16 * ktiles
  double* C;
  int64_t ldc;
  int c_row0, c_col0;
  int tiles_m, tiles_n;
  int lower;  // enumerate only tm >= tn (square tiles required)
  // gram epilogue
  const double* norm_a;
  const double* norm_b;
  int valid_a, valid_b;  // rows beyond these are padding (identity / zero)
  double denom;          // (2*sigma)*sigma, kernel.cpp:55
  double neg_inv_denom;  // -1 / denom (the epilogue multiplies; see below)
  const int* abort_flag; // per-part NPD flag: skip work once a pivot failed
  int mirror;            // G_GRAM_SYM: 1 = also write the upper triangle (public gram API);
                         // 0 = lower tiles only (the pipeline's K: nothing reads the upper half)
  // G_STORE (panel TRSM) with the forward substitution fused into the factorization:
  // fw[row] -= (C row) . fz over the tile's 128 columns, rows indexed like C (null: off)
  const double* fz;
  double* fw;
};

constexpr int kBK = 16;        // f64 per k-tile row = 128 B (one swizzle row)
constexpr int kBN = 128;
constexpr int kConsumerWarps = 8;
constexpr int kGemmThreads = (kConsumerWarps + 1) * 32;
constexpr int kStages = 4;


// BM = 32 (latency-bound panel steps: twice the CTAs of BM = 64) still loads a
// 64-row A box (the TMA box height); only its first 32 rows are used.
template <int BM>
struct GemmCfg {
  static constexpr int A_ROWS = BM < 64 ? 64 : BM;
  static constexpr int A_BYTES = A_ROWS * kBK * 8;
  static constexpr int B_BYTES = kBN * kBK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int WM = BM / 2;
  static constexpr int WN = kBN / 4;
  static constexpr int MT = WM / 8;
  static constexpr int NT = WN / 8;
  static constexpr int SMEM = kStages * STAGE_BYTES + 1024 + 2 * kStages * 8 + 64;
};

__device__ __forceinline__ void lower_tile_coords(int b, int& tm, int& tn) {
  int t = static_cast<int>((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
  while ((t + 1) * (t + 2) / 2 <= b) ++t;
  while (t * (t + 1) / 2 > b) --t;
  tm = t;
  tn = b - t * (t + 1) / 2;
}

// The symmetric gram epilogue (exp + mirrored write) needs more registers than the
// 168 a 9-warp CTA gets (registers are allocated per 4-warp group): that mode runs
// 3 warpgroups -- producer warpgroup shrunk to 40 registers with setmaxnreg.dec, the
// two DMMA warpgroups grown to 232 -- like dsyrk_persistent_kernel.
template <int MODE>
constexpr int gemm_threads() {
  return MODE == G_GRAM_SYM ? 384 : kGemmThreads;
}

// The 64-row panel GEMMs (TRSM, column updates: K = 128..512, a few microseconds of
// mainloop) fit two CTAs per SM at <= 112 registers, so one CTA's prologue / epilogue
// overlaps the other's mainloop.
template <int BM, int MODE>
constexpr int gemm_min_blocks() {
  return BM <= 64 && (MODE == G_UPDATE || MODE == G_STORE) ? 2 : 1;
}

template <int BM, int MODE>
__global__ void __launch_bounds__(gemm_threads<MODE>(), gemm_min_blocks<BM, MODE>())
    dgemm_tn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    GemmParams p) {
  using Cfg = GemmCfg<BM>;
  constexpr bool kWG = MODE == G_GRAM_SYM;             // warpgroup-specialised layout
  constexpr int kProducerWarp = kWG ? 0 : kConsumerWarps;
  constexpr int kFirstConsumer = kWG ? 4 : 0;
  pdl_wait();
  if (p.abort_flag && *reinterpret_cast<const volatile int*>(p.abort_flag)) return;

  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * Cfg::STAGE_BYTES);
  uint64_t* empty = full + kStages;

  int tm, tn;
  if (p.lower) {
    lower_tile_coords(blockIdx.x, tm, tn);
  } else {
    tm = blockIdx.x % p.tiles_m;
    tn = blockIdx.x / p.tiles_m;
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int KT = p.ktiles;
  if (kWG && warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
  if (kWG ? warp < 4 : warp == kConsumerWarps) {
    // ---------------- TMA producer ----------------
    if (warp == kProducerWarp && lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      const int arow = p.a_row0 + tm * BM, brow = p.b_row0 + tn * kBN;
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % kStages;
        const uint32_t ph = (kt / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        unsigned char* sa = smem + s * Cfg::STAGE_BYTES;
        unsigned char* sb = sa + Cfg::A_BYTES;
        const int ka = p.a_k0 + kt * kBK, kb = p.b_k0 + kt * kBK;
#pragma unroll
        for (int h = 0; h < Cfg::A_ROWS / 64; ++h) tma_load_2d(sa + h * 8192, &tmA, ka, arow + h * 64, &full[s]);
#pragma unroll
        for (int h = 0; h < kBN / 64; ++h) tma_load_2d(sb + h * 8192, &tmB, kb, brow + h * 64, &full[s]);
      }
    }
    return;
  }

  // ---------------- DMMA consumers ----------------
  if (kWG) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int cwarp = warp - kFirstConsumer;
  const int wm = cwarp >> 2, wn = cwarp & 3;
  const int lr = lane >> 2, lk = lane & 3;
  // gram modes: the row norms the epilogue needs are loaded before the mainloop, so
  // their latency hides behind it (they were among the epilogue's top stalls)
  constexpr bool kGram = MODE == G_GRAM_SYM || MODE == G_GRAM_CROSS;
  double na[kGram ? Cfg::MT : 1], nb[kGram ? Cfg::NT : 1][2];
  if constexpr (kGram) {
    const int gi0 = tm * BM + (cwarp >> 2) * Cfg::WM + (lane >> 2), gj0 = tn * kBN + (cwarp & 3) * Cfg::WN + 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i) na[i] = __ldg(p.norm_a + gi0 + i * 8);
#pragma unroll
    for (int j = 0; j < Cfg::NT; ++j) {
      nb[j][0] = __ldg(p.norm_b + gj0 + j * 8);
      nb[j][1] = __ldg(p.norm_b + gj0 + j * 8 + 1);
    }
  }
  double acc[Cfg::MT][Cfg::NT][2];
#pragma unroll
  for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % kStages;
    const uint32_t ph = (kt / kStages) & 1;
    mbar_wait(&full[s], ph);
    // Deferred release of the previous stage: its LDS results have been consumed by
    // the DMMAs issued before this wait, so the reads are complete.  Releasing right
    // after the last LDS let the TMA refill race a still-queued LDS (seen as rare
    // wrong fragments when a co-resident CTA congested the LSU).
    if (kt > 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[(kt - 1) % kStages]);
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

  // ---------------- epilogues ----------------
  const int r0 = wm * Cfg::WM + lr;        // + i*8
  const int c0 = wn * Cfg::WN + 2 * lk;    // + j*8 + {0,1}
  if constexpr (MODE == G_UPDATE || MODE == G_STORE) {
    double* Cb = p.C + static_cast<int64_t>(p.c_row0 + tm * BM) * p.ldc + (p.c_col0 + tn * kBN);
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) {
        double2* dst = reinterpret_cast<double2*>(Cb + static_cast<int64_t>(r0 + i * 8) * p.ldc + c0 + j * 8);
        if constexpr (MODE == G_UPDATE) {
          double2 v = *dst;
          v.x -= acc[i][j][0];
          v.y -= acc[i][j][1];
          *dst = v;
        } else {
          *dst = make_double2(acc[i][j][0], acc[i][j][1]);
        }
      }
    if constexpr (MODE == G_STORE) {
      if (p.fz) {
        // right-looking forward substitution step of this panel: w_r -= L21[r, :] . z_panel,
        // per-thread partial over its columns, then the 4 lanes of a row, then the 4
        // column warps in a fixed order (deterministic)
        __shared__ double fred[4][BM];
        double zc[Cfg::NT][2];
#pragma unroll
        for (int j = 0; j < Cfg::NT; ++j) {
          zc[j][0] = p.fz[tn * kBN + c0 + j * 8];
          zc[j][1] = p.fz[tn * kBN + c0 + j * 8 + 1];
        }
#pragma unroll
        for (int i = 0; i < Cfg::MT; ++i) {
          double part = 0.0;
#pragma unroll
          for (int j = 0; j < Cfg::NT; ++j) part = fma(acc[i][j][1], zc[j][1], fma(acc[i][j][0], zc[j][0], part));
          part += __shfl_xor_sync(0xffffffffu, part, 1);
          part += __shfl_xor_sync(0xffffffffu, part, 2);
          if (lk == 0) fred[wn][r0 + i * 8] = part;
        }
        consumer_sync(kConsumerWarps * 32);
        if (cwarp * 32 + lane < BM) {
          const int r = cwarp * 32 + lane;
          const double sum = (fred[0][r] + fred[1][r]) + (fred[2][r] + fred[3][r]);
          double* w = p.fw + p.c_row0 + tm * BM + r;
          *w -= sum;
        }
      }
    }
  } else {
    // Gaussian kernel epilogue (kernel.cpp:52-56): dist2 = (n_a + n_b) - 2*dot,
    // clamp at 0, exp(-dist2 / ((2 s) s)).  Padding rows are identity (sym) / 0.
    const int gi0 = tm * BM, gj0 = tn * kBN;
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int gi = gi0 + r0 + i * 8, gj = gj0 + c0 + j * 8 + e;
          double v;
          if (gi >= p.valid_a || gj >= p.valid_b) {
            v = (MODE == G_GRAM_SYM && gi == gj) ? 1.0 : 0.0;
          } else if (MODE == G_GRAM_SYM && gi == gj) {
            v = 1.0;  // squared_norm and the self dot sum identical products: dist2 == 0
          } else {
            double dist2 = (na[i] + nb[j][e]) - 2.0 * acc[i][j][e];
            if (dist2 < 0.0) dist2 = 0.0;
            // kernel.cpp:55 divides; a multiply by -1/denom moves the exponent by <= 1.5 ulp,
            // i.e. K by <= e^-1 |x| 2^-53 absolute -- far inside the 1e-13 K tolerance
            v = exp_nonpos(dist2 * p.neg_inv_denom);
          }
          acc[i][j][e] = v;
        }
    // direct write: K[gi][gj]; the symmetric diagonal tile keeps only gi >= gj
    double* Cb = p.C + static_cast<int64_t>(gi0) * p.ldc + gj0;
    const bool diag_tile = (MODE == G_GRAM_SYM) && (tm == tn);
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::NT; ++j) {
        const int r = r0 + i * 8, c = c0 + j * 8;
        double* dst = Cb + static_cast<int64_t>(r) * p.ldc + c;
        if (!diag_tile || r >= c + 1) {
          *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else if (r == c) {
          dst[0] = acc[i][j][0];
        }
      }
    if (MODE == G_GRAM_SYM && p.mirror) {
      // mirrored write K[gj][gi] = K[gi][gj] through a transposed smem stage
      // (coalesced rows; bitwise symmetric like kernel.cpp:113-116)
      double* T = reinterpret_cast<double*>(smem);  // pipeline ring is drained
      constexpr int TS = BM + 1;
      consumer_sync(kConsumerWarps * 32);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
#pragma unroll
        for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int c = c0 + j * 8 + e;
              if ((c >> 6) == half) T[(c & 63) * TS + r0 + i * 8] = acc[i][j][e];
            }
        consumer_sync(kConsumerWarps * 32);
        for (int cc = cwarp; cc < 64; cc += kConsumerWarps) {
          const int c = half * 64 + cc;
          double* dst = p.C + static_cast<int64_t>(gj0 + c) * p.ldc + gi0;
          for (int r = lane; r < BM; r += 32)
            if (tm != tn || r > c) dst[r] = T[cc * TS + r];
        }
        consumer_sync(kConsumerWarps * 32);
      }
    }
  }
}

}  // namespace pk
