// Microbenchmark of the centroid chain kernel (means_kernel): one cluster of n rows
// (k = 1) and k clusters of n/k rows, d = 90; prints us per launch and the chain bound.
#include <cstdio>
#include <vector>
#include "../paper_1805_00569_b200/csrc/kernels.cu"
using namespace pk;
__global__ void spin(long long cycles, long long* out) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  *out = clock64() - t0;
}
int main() {
  const int64_t n = 65536, d = 90;
  std::vector<double> X(n * d);
  for (size_t i = 0; i < X.size(); ++i) X[i] = 0.001 * (i % 977);
  double *dX, *dC;
  int64_t *mem, *st, *sz;
  cudaMalloc(&dX, X.size() * 8);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&dC, 64 * d * 8);
  std::vector<int64_t> m(n);
  for (int64_t i = 0; i < n; ++i) m[i] = i;
  cudaMalloc(&mem, n * 8);
  cudaMemcpy(mem, m.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&st, 64 * 8);
  cudaMalloc(&sz, 64 * 8);
  Counter c;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int k : {1, 8}) {
    std::vector<int64_t> s(k), z(k);
    for (int j = 0; j < k; ++j) {
      s[j] = j * (n / k);
      z[j] = n / k;
    }
    cudaMemcpy(st, s.data(), k * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(sz, z.data(), k * 8, cudaMemcpyHostToDevice);
    for (int w = 0; w < 3; ++w) launch_means(dX, d, mem, st, sz, k, dC, 0, c);
    cudaEventRecord(a);
    for (int w = 0; w < 10; ++w) launch_means(dX, d, mem, st, sz, k, dC, 0, c);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("k=%d rows/cluster=%lld: %.1f us per launch (chain bound at 8.2 cyc/row, 1.965 GHz: %.1f us)\n", k,
           (long long)(n / k), 1e3 * ms / 10, (n / k) * 8.2 / 1965.0);
  }
  long long* dcyc;
  cudaMalloc(&dcyc, 8);
  spin<<<1, 1>>>(1000000, dcyc);
  cudaEventRecord(a);
  spin<<<1, 1>>>(20000000, dcyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("SM clock while one CTA spins: %.0f MHz\n", 20000000 / (ms * 1e3));
  return 0;
}
