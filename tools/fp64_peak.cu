// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Produces the FP64 roofline denominators used in DESIGN.md / bench.py.
#include <cstdio>
#include <cuda_runtime.h>

#define CHK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dexp_loop(double* out, int iters) {
  double x = -1e-3 * threadIdx.x, s = 0.0;
  for (int it = 0; it < iters; ++it) { s += exp(x); x -= 1e-7; }
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CHK(cudaGetDevice(&dev));
  CHK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CHK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; CHK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps, threads = 32 * wpb, iters = 4000;
      dmma_loop<8><<<blocks, threads>>>(out, 100);
      CHK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_loop<8><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      CHK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256.0 * 8 * iters * (double)blocks * wpb;
      printf(", \"dmma_w%d_b%d_tflops\": %.3f", wpb, bps, flops / ms / 1e9);
    }
  }
  for (int bps : {2, 4, 8}) {
    int blocks = sms * bps, threads = 256, iters = 4000;
    dfma_loop<8><<<blocks, threads>>>(out, 100);
    CHK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<8><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    CHK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf(", \"dfma_b%d_tflops\": %.3f", bps, flops / ms / 1e9);
  }
  {
    int blocks = sms * 4, threads = 256, iters = 2000;
    dexp_loop<<<blocks, threads>>>(out, 10);
    CHK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dexp_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    CHK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"dexp_gexp_per_s\": %.3f", (double)iters * blocks * threads / ms / 1e6);
  }
  printf("}\n");
  return 0;
}
