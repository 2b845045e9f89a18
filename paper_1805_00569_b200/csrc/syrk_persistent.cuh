// syrk_persistent.cuh -- the Cholesky trailing update A22 -= L21 L21^T as a
// persistent FP64 tensor-core kernel (one CTA per SM, lower 128x128 tiles
// round-robin).  Per tile: DMMA mainloop over the 128-wide panel fed by a
// 3-stage TMA ring, while the producer warp TMA-prefetches the 128 KB C tile
// into shared memory; the epilogue subtracts in shared memory and writes the
// tile back with a TMA bulk store, so C never costs exposed HBM latency.
#pragma once

#include "gemm_dmma.cuh"

namespace pk {

struct SyrkParams {
  int row0;    // first trailing row/col (tiles start here)
  int k0;      // panel column origin
  int ktiles;  // panel width / 16
  int T;       // trailing tiles per side (lower tiles: T(T+1)/2)
  const int* abort_flag;
  int narrow;  // 0: all lower tiles; > 0: only tile columns tn < narrow (lookahead panel update)
};

__host__ __device__ __forceinline__ int syrk_tile_count(int T, int narrow) {
  if (narrow <= 0 || narrow >= T) return T * (T + 1) / 2;
  return narrow * (narrow + 1) / 2 + (T - narrow) * narrow;
}

constexpr int kSyrkStages = 3;
constexpr int kSyrkThreads = 384;  // warpgroup 0: TMA producer; warpgroups 1-2: DMMA consumers
constexpr int kSyrkStageBytes = (128 + 128) * kBK * 8;  // 32 KB
constexpr int kCBytes = 128 * 128 * 8;                  // 128 KB
constexpr int kSyrkSmem = kSyrkStages * kSyrkStageBytes + kCBytes + 1024 + 256;

// element (r, c) of a 128x128 f64 C tile staged as 16 TMA boxes {16 cols x 64 rows},
// box (c/16, r/64) at ((c/16)*2 + r/64) * 8 KB, 128B-swizzled inside the box
__device__ __forceinline__ uint32_t c_off(int r, int c) {
  return static_cast<uint32_t>((((c >> 4) * 2 + (r >> 6)) << 13)) + swz128(r & 63, c & 15);
}

__global__ void __launch_bounds__(kSyrkThreads, 1)
    dsyrk_persistent_kernel(const __grid_constant__ CUtensorMap tmA, SyrkParams p) {
  pdl_wait();
  if (p.abort_flag && *reinterpret_cast<const volatile int*>(p.abort_flag)) return;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* ring = smem;
  unsigned char* cbuf = smem + kSyrkStages * kSyrkStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(cbuf + kCBytes);
  uint64_t* empty = full + kSyrkStages;
  uint64_t* cfull = empty + kSyrkStages;
  uint64_t* cempty = cfull + 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSyrkStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    mbar_init(cfull, 1);
    mbar_init(cempty, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int ntiles = syrk_tile_count(p.T, p.narrow);
  const int KT = p.ktiles;
  // tile b -> (tm, tn): the lower triangle, or its first `narrow` tile columns
  auto coords = [&](int b, int& tm, int& tn) {
    const int tri = p.narrow * (p.narrow + 1) / 2;
    if (p.narrow <= 0) {
      // Bands of kBand tile rows; inside a band, blocks of kBand tile columns, row-major in a
      // block: the ~148 tiles in flight span 8 A-panel rows and ~19 B-panel rows (2 MB each at
      // K = 2048: L2-resident) instead of one tile row and every B panel -- in plain row-major
      // order each tile row re-streamed all the B panels from HBM (17.4 GB per launch at T = 145
      // against 3.1 GB compulsory) -- and consecutive tiles are neighbours in a row of C.
      constexpr int kBand = 8;
      int r, c;
      lower_tile_coords(b, r, c);
      const int R0 = r / kBand * kBand;
      const int nrows = p.T - R0 < kBand ? p.T - R0 : kBand;
      int q = b - R0 * (R0 + 1) / 2;            // index inside the band
      const int nblk = R0 / kBand;              // full blocks: columns [0, R0)
      if (q < nblk * kBand * nrows) {
        const int blk = q / (kBand * nrows), rq = q % (kBand * nrows);
        tm = R0 + rq / kBand;
        tn = blk * kBand + rq % kBand;
      } else {
        // the band's own triangle: columns R0 .. R0 + nrows - 1, rows >= column (row-major)
        q -= nblk * kBand * nrows;
        int i = 0;
        while (q > i) {
          q -= i + 1;
          ++i;
        }
        tm = R0 + i;
        tn = R0 + q;
      }
    } else if (b < tri) {
      lower_tile_coords(b, tm, tn);
    } else {
      tm = p.narrow + (b - tri) / p.narrow;
      tn = (b - tri) % p.narrow;
    }
  };

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 0 && lane == 0) {
      prefetch_tmap(&tmA);
      uint32_t g = 0;  // global k-step counter across tiles
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        int tm, tn;
        coords(tile, tm, tn);
        const int arow = p.row0 + tm * 128, brow = p.row0 + tn * 128;
        for (int kt = 0; kt < KT; ++kt, ++g) {
          const int s = g % kSyrkStages;
          const uint32_t ph = (g / kSyrkStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], kSyrkStageBytes);
          unsigned char* sa = ring + s * kSyrkStageBytes;
          unsigned char* sb = sa + 128 * kBK * 8;
          const int kc = p.k0 + kt * kBK;
          tma_load_2d(sa, &tmA, kc, arow, &full[s]);
          tma_load_2d(sa + 8192, &tmA, kc, arow + 64, &full[s]);
          tma_load_2d(sb, &tmA, kc, brow, &full[s]);
          tma_load_2d(sb + 8192, &tmA, kc, brow + 64, &full[s]);
          if (kt == (KT < kSyrkStages ? KT - 1 : kSyrkStages - 1)) {
            // C tile of this output block: wait until the previous tile's store drained
            mbar_wait(cempty, (it & 1) ^ 1);
            mbar_arrive_expect_tx(cfull, kCBytes);
            const uint64_t pol = l2_policy_evict_first();  // C is streamed once per group
            for (int cb = 0; cb < 8; ++cb)
              for (int rb = 0; rb < 2; ++rb)
                tma_load_2d_hint(cbuf + ((cb * 2 + rb) << 13), &tmA, p.row0 + tn * 128 + cb * 16,
                                 p.row0 + tm * 128 + rb * 64, cfull, pol);
          }
        }
      }
    }
    return;
  }

  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  const int cw = warp - 4;
  const int wm = cw >> 2, wn = cw & 3;
  const int lr = lane >> 2, lk = lane & 3;
  // fragment row -> tile row permutation: lanes 0-15 read tile rows {0,2,4,6},
  // lanes 16-31 rows {1,3,5,7}, so each half-warp of an LDS.64 touches 8 distinct
  // 16-byte chunks of the 128B-swizzled rows (conflict-free); the same
  // permutation on the B rows permutes the output columns (undone in the epilogue)
  const int pr = ((lr & 3) << 1) | (lr >> 2);
  int pc[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int n = 2 * lk + e;
    pc[e] = ((n & 3) << 1) | (n >> 2);
  }
  uint32_t g = 0;
  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    int tm, tn;
    coords(tile, tm, tn);
    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < KT; ++kt, ++g) {
      const int s = g % kSyrkStages;
      const uint32_t ph = (g / kSyrkStages) & 1;
      mbar_wait(&full[s], ph);
      if (g > 0) {  // deferred release of the previous stage (see dgemm_tn_kernel)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[(g - 1) % kSyrkStages]);
      }
      const unsigned char* sa = ring + s * kSyrkStageBytes;
      const unsigned char* sb = sa + 128 * kBK * 8;
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        const int k = ks * 4 + lk;
        double af[8], bf[4];
#pragma unroll
        for (int i = 0; i < 8; ++i) af[i] = lds_f64(sa, swz128(wm * 64 + i * 8 + pr, k));
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = lds_f64(sb, swz128(wn * 32 + j * 8 + pr, k));
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
    }
    // epilogue: C (smem) -= acc, then TMA store
    mbar_wait(cfull, it & 1);
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = wm * 64 + i * 8 + pr, c = wn * 32 + j * 8 + pc[e];
          const uint32_t q = smem_u32(cbuf) + c_off(r, c);
          sts_f64(q, lds_f64_at(q) - acc[i][j][e]);
        }
    fence_proxy_async();
    consumer_sync(kConsumerWarps * 32);
    if (threadIdx.x == 128) {
      const uint64_t pol = l2_policy_evict_first();
      for (int cb = 0; cb < 8; ++cb)
        for (int rb = 0; rb < 2; ++rb)
          tma_store_2d_hint(&tmA, p.row0 + tn * 128 + cb * 16, p.row0 + tm * 128 + rb * 64,
                            cbuf + ((cb * 2 + rb) << 13), pol);
      bulk_commit();
      bulk_wait_read0();
      mbar_arrive(cempty);
    }
  }
  if (threadIdx.x == 128) bulk_wait_read0();
}

}  // namespace pk
