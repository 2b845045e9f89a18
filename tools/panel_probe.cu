// Cycle cost of the dataflow chain's building blocks in isolation (one CTA):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/panel_probe tools/panel_probe.cu -lcuda
#include "../paper_1805_00569_b200/csrc/kernels.cu"
#include <cstdlib>
#include <vector>

__device__ long long g_probe[16];

__global__ void __launch_bounds__(256, 1) probe_kernel(const double* A) {
  extern __shared__ double sm[];
  double* S = sm;                      // [64][kDS]
  double* X = S + 64 * pk::kDS;        // [64][kDS]
  double* ds = X + 64 * pk::kDS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, lr = lane >> 2, lk = lane & 3;
  long long t[12] = {};
  for (int rep = 0; rep < 4; ++rep) {
    for (int e = tid; e < 64 * 64; e += 256) {
      S[(e / 64) * pk::kDS + e % 64] = A[e];
      X[(e / 64) * pk::kDS + e % 64] = (e / 64 == e % 64) ? 1.0 : 0.0;
    }
    __syncthreads();
    t[0] = clock64();
    if (warp == 0) pk::warp_diag32<pk::kDS>(pk::smem_u32(S), pk::smem_u32(X), pk::smem_u32(ds), lane);
    __syncthreads();
    t[1] = clock64();
    if (warp == 0) pk::warp_diag32u<pk::kDS>(pk::smem_u32(S + 32), pk::smem_u32(X + 32), pk::smem_u32(ds), lane);
    __syncthreads();
    t[2] = clock64();
    // one df_rn8 per warp on 4 warps (L10 = D10 X00 shape)
    if (warp >= 1 && warp <= 4) pk::df_rn8(S + (32 + 8 * (warp - 1)) * pk::kDS, S + (32 + 8 * (warp - 1)) * pk::kDS, X, 0, lr, lk);
    __syncthreads();
    t[3] = clock64();
    // one df_rn8 on one warp
    if (warp == 1) pk::df_rn8(S + 32 * pk::kDS, S + 32 * pk::kDS, X, 0, lr, lk);
    __syncthreads();
    t[4] = clock64();
    // 8 df_rn8 over 8 warps
    pk::df_rn8(S + 8 * warp * pk::kDS + 32, S + 8 * warp * pk::kDS + 32, X, 0, lr, lk);
    __syncthreads();
    t[5] = clock64();
    __syncthreads();
    t[6] = clock64();
  }
  if (tid == 0)
    for (int i = 0; i < 6; ++i) g_probe[i] = t[i + 1] - t[i];
}

int main() {
  const int m = 64;
  std::vector<double> A(m * m);
  srand(1);
  std::vector<double> G(m * m);
  for (auto& v : G) v = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double acc = i == j ? m : 0.0;
      for (int t = 0; t < m; ++t) acc += G[t * m + i] * G[t * m + j];
      A[i * m + j] = acc;
    }
  double* dA;
  cudaMalloc(&dA, m * m * 8);
  cudaMemcpy(dA, A.data(), m * m * 8, cudaMemcpyHostToDevice);
  const int smem = (2 * 64 * pk::kDS + 32 * 32) * 8;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 256, smem>>>(dA);
  cudaDeviceSynchronize();
  long long r[16];
  cudaMemcpyFromSymbol(r, g_probe, sizeof(r));
  printf("cycles: diag32 rolled %lld, diag32 unrolled %lld, 4x df_rn8 %lld, 1x df_rn8 %lld, 8x df_rn8 %lld, "
         "bare __syncthreads %lld (%s)\n",
         r[0], r[1], r[2], r[3], r[4], r[5], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
