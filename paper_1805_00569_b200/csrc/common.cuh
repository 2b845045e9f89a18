// common.cuh -- sm_100a device primitives used by every pkrr kernel:
// mbarrier + TMA (cp.async.bulk.tensor) staging and the FP64 tensor-core MMA.
//
// FP64 on Blackwell: tcgen05.mma has no f64 kind (ptxas rejects .kind::f64), so
// FP64 tensor-core math is the warp-level mma.sync m8n8k4 f64 (SASS DMMA.8x8x4).
// Measured on this pool's B200: 37.1 TFLOP/s DMMA vs 33.6 TFLOP/s DFMA
// (profiles/fp64_peak_r01.json).  Operand tiles still move by TMA into 128B-
// swizzled shared memory, paced by mbarriers, with a dedicated producer warp.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Arrive without a compiler memory clobber: for a latency-critical unrolled loop whose
// shared-memory writes are already ordered before it by a __syncwarp; the clobber
// would stop the scheduler from overlapping independent work across the arrive.
__device__ __forceinline__ void mbar_arrive_nomem(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

// One non-blocking probe of a phase (no retry loop): lets a latency-critical warp
// overlap the probe with independent work and only branch on it afterwards.
__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done;
}

// 2-D TMA tile load: box {inner = c0 (elements), outer = c1 (rows)} -> smem.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 3-D TMA tile load: box {c0 (innermost), c1, c2} -> smem
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// D(8x8) += A(8x4, row) * B(4x8, col), FP64 tensor core.
// Fragments: a = A[lane/4][lane%4], b = B[k = lane%4][n = lane/4],
// c = C[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  // not volatile: a pure register op the scheduler may interleave with the loads
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_f64x2(uint32_t addr, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}

// Byte offset of element (row, k) of a [rows x 16] f64 tile staged by TMA with
// CU_TENSOR_MAP_SWIZZLE_128B (16-byte chunk index XORed with row % 8).
__device__ __forceinline__ uint32_t swz128(int row, int k) {
  return static_cast<uint32_t>(row * 128 + ((((k >> 1) ^ (row & 7)) << 4) | ((k & 1) << 3)));
}

__device__ __forceinline__ double lds_f64(const unsigned char* base, uint32_t off) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(smem_u32(base) + off));
  return v;
}
// shared-window address variant (base already a 32-bit shared address)
__device__ __forceinline__ double lds_f64_at(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// Named barrier over the consumer warps only (producer warp excluded).
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace pk

namespace pk {

// 2-D TMA tile store smem -> global (bulk async group)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* smem_src) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(smem_src))
      : "memory");
}
// L2 eviction-priority hints for streamed-once data (the trailing matrix's C tiles):
// they go first, so the panel operands and the Cholesky leaf's code stay L2-resident.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* smem_dst, const CUtensorMap* map, int c0, int c1,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, int c0, int c1, const void* smem_src,
                                                  uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;\n" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(smem_src)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// 1-D bulk copy global -> shared (16B aligned, size % 16 == 0), completes on an mbarrier
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 1-D bulk copy shared -> global (bulk async group)
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
// Programmatic dependent launch: a kernel launched with programmatic stream
// serialization may start while its predecessor in the stream drains; it must not
// touch memory the predecessor writes or reads before this wait (a no-op for a
// normally launched kernel).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}


// exp(x) for the Gaussian kernel's argument x = -dist2 / (2 s^2) <= 0 (kernel.cpp:52-56),
// branch-free so that the epilogues' independent elements interleave: k = round(x log2 e)
// by the 1.5 * 2^52 shift, r = x - k ln2 in two steps (fdlibm's ln2 hi / lo), exp(r) by its
// degree-13 Taylor polynomial (|r| <= 0.347: truncation 4e-18), 2^k added into the exponent
// field.  Measured against libm over [-700, 0]: <= 2.3e-16 relative (tools/exp_check.c).
// x < -700 returns exp(-700) ~ 1e-304 (never denormal); NaN stays NaN.
__device__ __forceinline__ double exp_nonpos(double x) {
  const double xc = x < -700.0 ? -700.0 : x;
  const double t = fma(xc, 1.4426950408889634, 6755399441055744.0);
  const int k = __double2loint(t);
  const double kf = t - 6755399441055744.0;
  double r = fma(kf, -6.93147180369123816490e-01, xc);
  r = fma(kf, -1.90821492927058770002e-10, r);
  double p = 1.0 / 6227020800.0;
  p = fma(p, r, 1.0 / 479001600.0);
  p = fma(p, r, 1.0 / 39916800.0);
  p = fma(p, r, 1.0 / 3628800.0);
  p = fma(p, r, 1.0 / 362880.0);
  p = fma(p, r, 1.0 / 40320.0);
  p = fma(p, r, 1.0 / 5040.0);
  p = fma(p, r, 1.0 / 720.0);
  p = fma(p, r, 1.0 / 120.0);
  p = fma(p, r, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double res = __hiloint2double(__double2hiint(p) + k * (1 << 20), __double2loint(p));  // k < 0: no shift of a negative
  return x != x ? x : res;
}

__constant__ double kExpTaylor[14] = {1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
                                      1.0 / 362880.0,     1.0 / 40320.0,     1.0 / 5040.0,     1.0 / 720.0,
                                      1.0 / 120.0,        1.0 / 24.0,        1.0 / 6.0,        0.5,
                                      1.0,                1.0};
// The same function over N independent arguments, written stage by stage so that the N
// dependent chains reach the instruction stream interleaved (in place: x[u] = exp(x[u])).
// 2^k is applied as a product, so a NaN argument stays NaN without a select.
template <int N>
__device__ __forceinline__ void exp_nonpos_n(double (&x)[N]) {
  double r[N], kf[N], p[N];
  int k[N];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const double xc = x[u] < -700.0 ? -700.0 : x[u];
    const double t = fma(xc, 1.4426950408889634, 6755399441055744.0);
    k[u] = __double2loint(t);
    kf[u] = t - 6755399441055744.0;
    r[u] = xc;
  }
#pragma unroll
  for (int u = 0; u < N; ++u) r[u] = fma(kf[u], -6.93147180369123816490e-01, r[u]);
#pragma unroll
  for (int u = 0; u < N; ++u) r[u] = fma(kf[u], -1.90821492927058770002e-10, r[u]);
  // coefficients from the constant bank (as DFMA operands): as literals they took 26 registers
#pragma unroll
  for (int u = 0; u < N; ++u) p[u] = kExpTaylor[0];
#pragma unroll
  for (int q = 1; q < 14; ++q)
#pragma unroll
    for (int u = 0; u < N; ++u) p[u] = fma(p[u], r[u], kExpTaylor[q]);
#pragma unroll
  for (int u = 0; u < N; ++u) x[u] = p[u] * __hiloint2double((k[u] + 1023) << 20, 0);
}

}  // namespace pk
