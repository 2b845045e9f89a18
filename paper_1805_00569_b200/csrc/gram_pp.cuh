// gram_pp.cuh -- the pipeline's symmetric Gaussian kernel matrix K (lower tiles) as a
// persistent "ping-pong" DMMA kernel (kernel.cpp:52-56, 81-119; the gram half of
// strategies.cpp:284-294 runs through dgemm_tn_kernel<G_GRAM_CROSS>).
//
// dgemm_tn_kernel<128, G_GRAM_SYM> runs one 128 x 128 tile per CTA: its short mainloop
// (K = dp = 96 at d = 90: 6 k-tiles) is followed by the exp / store epilogue with the
// DMMA pipe idle, and the next tile's CTA starts only after that (one CTA per SM): the
// tensor pipe was ~52 % busy (profiles/ncu_gram_r01.txt).  Here each SM runs one
// persistent CTA with TWO DMMA warpgroups that take alternate 128 x 64 half-tiles of the
// CTA's share, each fed by its own TMA producer thread and 4-stage ring (one shared ring
// aliased barrier phases once a tile's k-tiles outnumbered the stages); warpgroup 1
// starts after warpgroup 0's first mainloop, so while one warpgroup evaluates
// exp(-d^2 / ((2 s) s)) and stores its half-tile, the other runs its mainloop.  Same
// arithmetic per element as G_GRAM_SYM (bitwise the same K).
#pragma once

#include <type_traits>

#include "gemm_dmma.cuh"

namespace pk {

constexpr int kPPStages = 4;           // per warpgroup ring
constexpr int kPPA = 128 * kBK * 8;      // A: 128 rows x 16 (two 64-row TMA boxes)
constexpr int kPPB = 64 * kBK * 8;       // B: 64 rows x 16
constexpr int kPPStage = kPPA + kPPB;    // 24 KB
constexpr int kPPThreads = 384;          // producer warpgroup + 2 DMMA warpgroups
constexpr int kPPSmem = 2 * kPPStages * kPPStage + 1024 + 4 * kPPStages * 8 + 64;

struct GramPPParams {
  int T;          // 128-row tiles per side
  int ktiles;     // dp / 16
  double* K;
  int64_t ldk;
  const double* norms;
  int valid;      // rows >= valid are padding (identity)
  double neg_inv_denom;
  const int* abort_flag;
  double* A;      // != null: also A = K + shift I (the first lambda's system: no assemble pass)
  double shift;
  int turns;      // strict alternation of the warpgroups' mainloops (short mainloops: small d)
};

__global__ void __launch_bounds__(kPPThreads, 1)
    gram_pp_kernel(const __grid_constant__ CUtensorMap tmX, GramPPParams p) {
  pdl_wait();
  if (p.abort_flag && *reinterpret_cast<const volatile int*>(p.abort_flag)) return;
  extern __shared__ unsigned char pp_smem_raw[];
  unsigned char* smem = pp_smem_raw + ((1024u - (smem_u32(pp_smem_raw) & 1023u)) & 1023u);
  uint64_t* fullb = reinterpret_cast<uint64_t*>(smem + 2 * kPPStages * kPPStage);  // [2][S]
  uint64_t* emptyb = fullb + 2 * kPPStages;                                          // [2][S]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nhalf = p.T * (p.T + 1);  // lower 128-tiles x 2 column halves
  const int KT = p.ktiles;
  if (tid == 0) {
    for (int s = 0; s < 2 * kPPStages; ++s) {
      mbar_init(&fullb[s], 1);
      mbar_init(&emptyb[s], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp < 2 && lane == 0) {
      // producer of warpgroup `warp`: its half-tiles t = warp, warp + 2, ... in order
      const int w = warp;
      unsigned char* ring = smem + w * kPPStages * kPPStage;
      uint64_t* full = fullb + w * kPPStages;
      uint64_t* empty = emptyb + w * kPPStages;
      prefetch_tmap(&tmX);
      int g = 0;
      for (int t = w;; t += 2) {
        const int idx = blockIdx.x + t * gridDim.x;
        if (idx >= nhalf) break;
        int I, J;
        lower_tile_coords(idx >> 1, I, J);
        const int row0 = I * 128, col0 = J * 128 + (idx & 1) * 64;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % kPPStages;
          mbar_wait(&empty[s], ((g / kPPStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], kPPStage);
          unsigned char* sa = ring + s * kPPStage;
          tma_load_2d(sa, &tmX, 16 * kt, row0, &full[s]);
          tma_load_2d(sa + 8192, &tmX, 16 * kt, row0 + 64, &full[s]);
          tma_load_2d(sa + kPPA, &tmX, 16 * kt, col0, &full[s]);
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int wg = (warp - 4) >> 2, cw = (warp - 4) & 3;
  const int wm = cw >> 1, wn = cw & 1;  // 2 x 2 warps, 64 x 32 each
  const int lr = lane >> 2, lk = lane & 3;
  const unsigned char* ring = smem + wg * kPPStages * kPPStage;
  uint64_t* full = fullb + wg * kPPStages;
  uint64_t* empty = emptyb + wg * kPPStages;
  // Strict alternation of the two warpgroups' mainloops (named barriers 8 + wg, 256
  // threads: the waiting warpgroup syncs, the other arrives when its mainloop is done):
  // left alone they drifted into running both mainloops, then both epilogues, together --
  // the DMMA pipe idle through the latter.  Warpgroup 1 primes warpgroup 0's first turn.
  auto turn_wait = [&] { asm volatile("bar.sync %0, 256;\n" ::"r"(8 + wg) : "memory"); };
  auto turn_pass = [&] { asm volatile("bar.arrive %0, 256;\n" ::"r"(8 + (wg ^ 1)) : "memory"); };
  const bool turns = p.turns != 0;
  if (turns && wg == 1) turn_pass();
  int g = 0;
  for (int t = wg;; t += 2) {
    const int idx = blockIdx.x + t * gridDim.x;
    if (idx >= nhalf) break;
    int I, J;
    lower_tile_coords(idx >> 1, I, J);
    const int row0 = I * 128, col0 = J * 128 + (idx & 1) * 64;
    // the norms the epilogue needs, loaded ahead of the mainloop
    double na[8], nb[4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) na[i] = __ldg(p.norms + row0 + wm * 64 + i * 8 + lr);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      nb[j][0] = __ldg(p.norms + col0 + wn * 32 + j * 8 + 2 * lk);
      nb[j][1] = __ldg(p.norms + col0 + wn * 32 + j * 8 + 2 * lk + 1);
    }
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (turns) turn_wait();
    for (int kt = 0; kt < KT; ++kt, ++g) {
      const int s = g % kPPStages;
      mbar_wait(&full[s], (g / kPPStages) & 1);
      if (kt > 0) {  // deferred release (see gemm_dmma.cuh)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[(g - 1) % kPPStages]);
      }
      const unsigned char* sa = ring + s * kPPStage;
      const unsigned char* sb = sa + kPPA;
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        const int k = ks * 4 + lk;
        double af[8], bf[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = lds_f64(sa, swz128(wm * 64 + i * 8 + lr, k));
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = lds_f64(sb, swz128(wn * 32 + j * 8 + lr, k));
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[(g - 1) % kPPStages]);
    if (turns) turn_pass();
    // epilogue (kernel.cpp:52-56): dist2 = (n_a + n_b) - 2 dot, clamp at 0,
    // exp(dist2 * -1/((2 s) s)); unit diagonal; padding identity; diagonal tiles keep
    // only gi >= gj (nothing reads their upper triangle)
    // Branch-free per element (selects only) and, off the diagonal tiles, no branch around
    // the stores either: a row's 8 exp chains sit in one basic block and interleave.  (With
    // two chains per block every dependent DFMA queued behind a 16-cycle DMMA of the other
    // warpgroup's mainloop on the shared FP64 datapath: the epilogue, not the mainloop, set
    // the alternation period.)
    auto epilogue = [&](auto diag_c) {
      constexpr bool kDiag = decltype(diag_c)::value;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int gi = row0 + wm * 64 + i * 8 + lr;
        double v[4][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // 4 chains at a time (register budget: 128 accumulator registers)
          double ex[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 2 * h + (u >> 1), e = u & 1;
            double dist2 = (na[i] + nb[j][e]) - 2.0 * acc[i][j][e];
            dist2 = dist2 < 0.0 ? 0.0 : dist2;
            ex[u] = dist2 * p.neg_inv_denom;
          }
          exp_nonpos_n<4>(ex);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 2 * h + (u >> 1), e = u & 1;
            const int gj = col0 + wn * 32 + j * 8 + 2 * lk + e;
            const bool pad = gi >= p.valid || gj >= p.valid;
            v[j][e] = gi == gj ? 1.0 : (pad ? 0.0 : ex[u]);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int gj = col0 + wn * 32 + j * 8 + 2 * lk;
          double* dst = p.K + static_cast<int64_t>(gi) * p.ldk + gj;
          if (!kDiag || gi >= gj + 1)
            *reinterpret_cast<double2*>(dst) = make_double2(v[j][0], v[j][1]);
          else if (gi == gj)
            dst[0] = v[j][0];
          if (p.A) {
            double* da = p.A + static_cast<int64_t>(gi) * p.ldk + gj;
            if (!kDiag || gi >= gj + 1)
              *reinterpret_cast<double2*>(da) =
                  make_double2(kDiag && gi == gj ? v[j][0] + p.shift : v[j][0], kDiag && gi == gj + 1 ? v[j][1] + p.shift : v[j][1]);
            else if (gi == gj)
              da[0] = v[j][0] + p.shift;
          }
        }
      }
    };
    if (I == J)
      epilogue(std::true_type{});
    else
      epilogue(std::false_type{});
  }
}

}  // namespace pk
