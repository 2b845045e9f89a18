// ozaki_syrk.cuh -- FP64-accurate Cholesky trailing update on the int8 tensor
// cores (tcgen05.mma kind::i8, TMEM accumulators): Ozaki-scheme splitting.
//
//   Each panel row i (K = 512 entries) gets a power-of-two scale 2^e_i with
//   max|x| 2^-e_i < 1/2 and is split into S = 8 signed 7-bit slices,
//       x = 2^e_i * sum_{s=1..8} d_s 2^{-7 s},   |d_s| <= 64,
//   (55 significant bits).  Then
//       (L21 L21^T)_ij = 2^{e_i + e_j} sum_{g=2..9} 2^{-7 g} S_g(i,j),
//       S_g = sum_{s+t=g} D_s D_t^T   (exact int32: |S_g| <= 8*512*64*64 < 2^25).
//   Pairs with s + t > 9 are dropped (each < 2^-70 relative); the result has the
//   error of an FP64 GEMM (K * 2^-53 relative to the row norms).
//
// Kernel: one CTA per 128 x 64 output tile of the lower triangle.  Per 32-byte K
// stage the 8 A-slices (128 rows) and 8 B-slices (64 rows) are TMA-staged with a
// 32B swizzle; one elected thread issues the 36 tcgen05.mma (M128 N64 K32) of the
// stage into 8 TMEM accumulators (one per g, 64 columns each = all 512 columns);
// tcgen05.commit frees the stage.  The C tile (FP64) is TMA-prefetched during the
// mainloop; 4 epilogue warps read TMEM (tcgen05.ld), recombine in FP64, update C
// in shared memory and TMA-store it.
#pragma once

#include "common.cuh"

namespace pk {

constexpr int kOzS = 8;                       // slices
constexpr int kOzM = 128, kOzN = 64, kOzK = 32;  // tile and K per stage (int8)
constexpr int kOzStages = 3;
constexpr int kOzABytes = kOzS * kOzM * kOzK;  // 32 KB
constexpr int kOzBBytes = kOzS * kOzN * kOzK;  // 16 KB
constexpr int kOzStageBytes = kOzABytes + kOzBBytes;
constexpr int kOzCBytes = kOzM * kOzN * 8;     // 64 KB
constexpr int kOzSmem = kOzStages * kOzStageBytes + kOzCBytes + 1024 + 256;
constexpr int kOzThreads = 256;

struct OzParams {
  int row0;     // first row/col of A covered by the C tiles
  int R;        // trailing rows (multiple of 128)
  int ksteps;   // K / 32
  const int* exps;  // per sliced row: e_i
  const int* abort_flag;
  int srow;     // row of the slice / exps arrays that corresponds to row0 (lookahead (b): 128 G)
  int narrow;   // > 0: only the first `narrow` 64-column tiles (lookahead (a)); 0: whole triangle
};

__device__ __forceinline__ uint64_t oz_desc_sw32(uint32_t saddr) {
  // UMMA shared-memory descriptor, K-major, 32B swizzle: start (>>4), LBO = 1 (unused
  // for swizzled K-major), SBO = 8 rows * 32 B = 256 B (>>4 = 16), version 1 (sm_100),
  // layout type 6 = SWIZZLE_32B.
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(16) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(6) << 61);
}

// kind::i8 instruction descriptor: D = S32, A/B signed int8, K-major, N = 64, M = 128
constexpr uint32_t kOzIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((kOzN >> 3) << 17) | ((kOzM >> 4) << 24);

__device__ __forceinline__ void oz_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kOzIdesc), "r"(acc));
}

__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}

// 32 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// lower-triangle 128 x 64 tiles: row block I has 2I + 2 tiles (J = 0 .. 2I+1)
__device__ __forceinline__ void oz_tile_coords(int b, int& I, int& J) {
  int t = static_cast<int>((sqrt(4.0 * b + 1.0) - 1.0) * 0.5);
  while ((t + 1) * (t + 2) <= b) ++t;
  while (t * (t + 1) > b) --t;
  I = t;
  J = b - t * (t + 1);
}

// tmA8 / tmB8: the int8 slices as a 3-D tensor {K, R, 8} with boxes {32, 128, 8} /
// {32, 64, 8} (one TMA op stages all 8 slices of a stage); tmC: the FP64 matrix A
// (box {16, 64}, 128B swizzle, as for the DMMA kernels)
#ifdef OZ_TRACE
__device__ long long g_oz_trace[8][65536];
#define OZ_MARK(i) \
  if (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 128) g_oz_trace[i][blockIdx.x & 65535] = clock64();
#else
#define OZ_MARK(i)
#endif

__global__ void __launch_bounds__(kOzThreads, 1)
    ozaki_syrk_kernel(const __grid_constant__ CUtensorMap tmA8, const __grid_constant__ CUtensorMap tmB8,
                      const __grid_constant__ CUtensorMap tmC, OzParams p) {
  if (p.abort_flag && *reinterpret_cast<const volatile int*>(p.abort_flag)) return;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* ring = smem;
  unsigned char* cbuf = smem + kOzStages * kOzStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(cbuf + kOzCBytes);
  uint64_t* empty = full + kOzStages;
  uint64_t* cfull = empty + kOzStages;
  uint64_t* tfull = cfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  int I, J;
  if (p.narrow > 0) {  // the first `narrow` tile columns: the triangle of rows I < narrow/2, then full rows
    const int g2 = p.narrow >> 1, tri = g2 * (g2 + 1);
    if (static_cast<int>(blockIdx.x) < tri) {
      oz_tile_coords(blockIdx.x, I, J);
    } else {
      I = g2 + (blockIdx.x - tri) / p.narrow;
      J = (blockIdx.x - tri) % p.narrow;
    }
  } else {
    oz_tile_coords(blockIdx.x, I, J);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    OZ_MARK(0);
    for (int s = 0; s < kOzStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(cfull, 1);
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM: all 512 columns (8 accumulators x 64)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  const int KS = p.ksteps;
  if (threadIdx.x == 0) OZ_MARK(1);

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      prefetch_tmap(&tmA8);
      prefetch_tmap(&tmB8);
      prefetch_tmap(&tmC);
      // C tile: 4 column boxes (16 doubles) x 2 row boxes (64 rows)
      mbar_arrive_expect_tx(cfull, kOzCBytes);
      for (int cb = 0; cb < 4; ++cb)
        for (int rb = 0; rb < 2; ++rb)
          tma_load_2d(cbuf + ((cb * 2 + rb) << 13), &tmC, p.row0 + J * kOzN + cb * 16, p.row0 + I * kOzM + rb * 64,
                      cfull);
      for (int ks = 0; ks < KS; ++ks) {
        const int st = ks % kOzStages;
        const uint32_t ph = (ks / kOzStages) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], kOzStageBytes);
        unsigned char* sa = ring + st * kOzStageBytes;
        unsigned char* sb = sa + kOzABytes;
        tma_load_3d(sa, &tmA8, ks * kOzK, p.srow + I * kOzM, 0, &full[st]);
        tma_load_3d(sb, &tmB8, ks * kOzK, p.srow + J * kOzN, 0, &full[st]);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: the warp waits, one elected lane issues; descriptors are
    // base + compile-time offsets (start-address field, 16-byte units) ----
    const uint64_t dA0 = oz_desc_sw32(smem_u32(ring));
    const uint64_t dB0 = oz_desc_sw32(smem_u32(ring) + kOzABytes);
    for (int ks = 0; ks < KS; ++ks) {
      const int st = ks % kOzStages;
      const uint32_t ph = (ks / kOzStages) & 1;
      mbar_wait(&full[st], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t sa = dA0 + static_cast<uint64_t>((st * kOzStageBytes) >> 4);
        const uint64_t sb = dB0 + static_cast<uint64_t>((st * kOzStageBytes) >> 4);
        const uint32_t acc0 = ks > 0 ? 1u : 0u;
#pragma unroll
        for (int s = 0; s < kOzS; ++s)
#pragma unroll
          for (int t = 0; t < kOzS - s; ++t)
            oz_mma(tmem + (s + t) * kOzN, sa + ((s * kOzM * kOzK) >> 4), sb + ((t * kOzN * kOzK) >> 4),
                   s > 0 ? 1u : acc0);
        oz_commit(&empty[st]);  // frees the stage when these MMAs have read it
      }
      __syncwarp();
    }
    if (elect_one()) oz_commit(tfull);  // all accumulators complete
    __syncwarp();
    if (lane == 0 && threadIdx.x == 32) OZ_MARK(2);
  }
  // ---- epilogue (all 8 warps): TMEM -> FP64 recombination -> C (smem) -> TMA store.
  // warp w reads TMEM lane quarter w % 4, columns [32 (w / 4), +32) of each accumulator.
  {
    __syncwarp();
    const int q = warp & 3, ch = warp >> 2;
    const int r = q * 32 + lane;  // tile row
    mbar_wait(tfull, 0);
    tc_fence_after();
    if (threadIdx.x == 128) OZ_MARK(3);
    mbar_wait(cfull, 0);
    const double sci = __longlong_as_double(static_cast<long long>(1023 + p.exps[p.srow + I * kOzM + r]) << 52);
    double acc[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) acc[c] = 0.0;
#pragma unroll 1
    for (int g = kOzS - 1; g >= 0; --g) {  // smallest terms first
      int v[32];
      tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + g * kOzN + ch * 32, v);
      const double w = __longlong_as_double(static_cast<long long>(1023 - 7 * (g + 2)) << 52);  // 2^{-7(g+2)}
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[c] = fma(static_cast<double>(v[c]), w, acc[c]);
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int col = ch * 32 + c;
      const double scj = __longlong_as_double(static_cast<long long>(1023 + p.exps[p.srow + J * kOzN + col]) << 52);
      const uint32_t off = static_cast<uint32_t>((((col >> 4) * 2 + (r >> 6)) << 13)) + swz128(r & 63, col & 15);
      const uint32_t addr = smem_u32(cbuf) + off;
      sts_f64(addr, lds_f64_at(addr) - acc[c] * sci * scj);  // power-of-two scales: exact
    }
    fence_proxy_async();
    tc_fence_before();
    if (threadIdx.x == 128) OZ_MARK(4);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // producer tail: the tcgen05.commit arrivals on the last kOzStages 'empty'
    // barriers are asynchronous and not ordered with the 'tfull' arrival; wait until
    // they have landed so none is delivered into shared memory after this CTA exits
    // (it would corrupt whatever CTA the SM places there next).
    for (int ks = KS; ks < KS + kOzStages; ++ks) mbar_wait(&empty[ks % kOzStages], ((ks / kOzStages) & 1) ^ 1);
    for (int cb = 0; cb < 4; ++cb)
      for (int rb = 0; rb < 2; ++rb)
        tma_store_2d(&tmC, p.row0 + J * kOzN + cb * 16, p.row0 + I * kOzM + rb * 64, cbuf + ((cb * 2 + rb) << 13));
    bulk_commit();
    bulk_wait_read0();
    OZ_MARK(5);
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// ---- slicing: panel rows [row0, row0+R) x cols [k0, k0+K) of A -> int8 [8][R][K] + exps ----
__global__ void ozaki_slice_kernel(const double* __restrict__ A, int64_t lda, int row0, int k0, int R, int K,
                                   int8_t* __restrict__ slices, int* __restrict__ exps,
                                   const int* abort_flag, int Rstride) {
  if (abort_flag && *reinterpret_cast<const volatile int*>(abort_flag)) return;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= R) return;
  const double* row = A + static_cast<int64_t>(row0 + warp) * lda + k0;
  double mx = 0.0;
  for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(row[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int e = mx > 0.0 ? ilogb(mx) + 2 : 0;  // max|x| 2^-e < 1/2
  if (lane == 0) exps[warp] = e;
  for (int k = lane; k < K; k += 32) {
    double x = ldexp(row[k], -e);
#pragma unroll
    for (int s = 0; s < kOzS; ++s) {
      const double t = x * 128.0;
      const double d = rint(t);
      slices[(static_cast<int64_t>(s) * Rstride + warp) * K + k] = static_cast<int8_t>(d);
      x = t - d;
    }
  }
}

}  // namespace pk
