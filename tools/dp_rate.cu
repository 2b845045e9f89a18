// FP64 (non-tensor) issue rates on this GPU: independent DFMA, DADD, DMUL chains and the
// assign kernel's pattern (__dmul_rn then a dependent __dadd_rn per chain), 8 chains per
// thread, 148 x 8 CTAs of 256 threads.  Reports warp-instructions per cycle per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void kern(double* out, int iters, double a, double b) {
  double c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE == 0) c[q] = fma(c[q], a, b);
      if (MODE == 1) c[q] = __dadd_rn(c[q], b);
      if (MODE == 2) c[q] = __dmul_rn(c[q], a);
      if (MODE == 3) c[q] = __dadd_rn(c[q], __dmul_rn(a + q, b));
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += c[q];
  if (s == 12345.678) out[0] = s;
}

template <int MODE>
void run(const char* name, int per_iter) {
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  kern<MODE><<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<MODE><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_instr = double(blocks) * threads / 32 * iters * 8 * per_iter;
  const double cycles = ms * 1e-3 * 1.9e9;
  printf("%-22s %.3f ms  %.2f warp-instr / cycle / SM  (%.1f lane-ops / cycle / SM)\n", name, ms,
         warp_instr / cycles / 148, warp_instr * 32 / cycles / 148);
  cudaFree(out);
}

int main() {
  run<0>("DFMA", 1);
  run<1>("DADD", 1);
  run<2>("DMUL", 1);
  run<3>("DMUL+DADD", 2);
  return 0;
}
