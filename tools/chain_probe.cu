// One warp: DADD chain over values read from shared memory (64-row blocks, 32 lanes
// = 32 columns), no barriers: cycles per row for the centroid-chain inner loop.
#include <cstdio>
#include "../paper_1805_00569_b200/csrc/common.cuh"
using namespace pk;
template <int MODE>
__global__ void probe(double* out, long long* cyc, int blocks) {
  __shared__ double buf[2][64 * 32];
  __shared__ uint64_t bar, full[4], empty[4];
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= 32) {  // MODE 2: 7 warps spin on a barrier until the chain is done
    mbar_wait(&bar, 0);
    return;
  }
  for (int i = threadIdx.x; i < 2 * 64 * 32; i += 32) (&buf[0][0])[i] = 1e-3 * (i % 97);
  __syncwarp();
  double s = 0.0;
  const long long t0 = clock64();
  for (int b = 0; b < blocks; ++b) {
    const uint32_t base = smem_u32(&buf[b & 1][threadIdx.x]);
    if (MODE == 3) {  // + per-block barrier traffic like means_kernel (wait full, arrive empty)
      if (threadIdx.x == 0) mbar_arrive(&full[b & 3]);  // self-produced
      mbar_wait(&full[b & 3], (b >> 2) & 1);
      double v[64];
#pragma unroll
      for (int u = 0; u < 64; ++u) v[u] = lds_f64_at(base + u * 32 * 8);
#pragma unroll
      for (int u = 0; u < 64; ++u) s = __dadd_rn(s, v[u]);
      __syncwarp();
      if (threadIdx.x == 0) mbar_arrive(&empty[b & 3]);
    } else if (MODE == 0) {
      double v[64];
#pragma unroll
      for (int u = 0; u < 64; ++u) v[u] = lds_f64_at(base + u * 32 * 8);
#pragma unroll
      for (int u = 0; u < 64; ++u) s = __dadd_rn(s, v[u]);
    } else {
      const double* p = &buf[b & 1][threadIdx.x];
#pragma unroll
      for (int u = 0; u < 64; ++u) s = __dadd_rn(s, p[u * 32]);
    }
  }
  const long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) {
    *cyc = t1 - t0;
    mbar_arrive(&bar);
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 8);
  long long h;
  probe<0><<<1, 32>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("volatile LDS x64 then DADD x64: %.2f cycles/row\n", h / 64000.0);
  probe<1><<<1, 32>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("plain smem loads (compiler scheduled): %.2f cycles/row\n", h / 64000.0);
  probe<0><<<1, 256>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("volatile LDS, 7 other warps spinning on try_wait: %.2f cycles/row\n", h / 64000.0);
  probe<3><<<1, 32>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("with per-block wait(full)+arrive(empty): %.2f cycles/row\n", h / 64000.0);
}
