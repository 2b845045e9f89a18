// Dependent-chain latency of FP64 add / fma on this GPU: one thread, and one full warp.
#include <cstdio>
__global__ void chain(double* out, long long* cyc, int n, double x) {
  double s = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, x);
  long long t1 = clock64();
  double f = 1.0;
  for (int i = 0; i < n; ++i) f = fma(f, x, 0.5);
  long long t2 = clock64();
  out[threadIdx.x] = s + f;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 32); cudaMalloc(&c, 16);
  for (int threads : {1, 32}) {
    chain<<<1, threads>>>(o, c, 1000, 1.0000001);
    chain<<<1, threads>>>(o, c, 100000, 1.0000001);
    long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("%2d threads: dadd %.2f cycles/op, dfma %.2f cycles/op\n", threads, h[0] / 1e5, h[1] / 1e5);
  }
}
