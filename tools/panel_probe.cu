// Cycle cost of the dataflow chain's 32-column diagonal panel in isolation (one CTA):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/panel_probe tools/panel_probe.cu -lcuda
#include "../paper_1805_00569_b200/csrc/kernels.cu"
#include <cstdlib>
#include <vector>

__device__ long long g_probe[16];

__global__ void __launch_bounds__(288, 1) probe_kernel(const double* A) {
  extern __shared__ double sm[];
  double* S = sm;
  double* ds = S + 64 * pk::kDS;
  __shared__ uint64_t cbar[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int j = 0; j < 32; ++j) pk::mbar_init(&cbar[j], 1);
    pk::fence_mbar_init();
  }
  __syncthreads();
  long long t[8] = {};
  for (int rep = 0; rep < 4; ++rep) {
    for (int e = tid; e < 64 * 64; e += 288) S[(e / 64) * pk::kDS + e % 64] = A[e];
    __syncthreads();
    t[0] = clock64();
    if (warp == 0) pk::warp_diag32<pk::kDS>(pk::smem_u32(S), pk::smem_u32(S + 32 * pk::kDS), pk::smem_u32(ds), lane);
    __syncthreads();
    t[1] = clock64();
    for (int e = tid; e < 64 * 64; e += 288) S[(e / 64) * pk::kDS + e % 64] = A[e];
    __syncthreads();
    t[2] = clock64();
    if (warp == 0) pk::warp_diag32<pk::kDS>(pk::smem_u32(S), pk::smem_u32(S + 32 * pk::kDS), pk::smem_u32(ds), lane);
    __syncthreads();
    t[3] = clock64();
    for (int e = tid; e < 64 * 64; e += 288) S[(e / 64) * pk::kDS + e % 64] = A[e];
    __syncthreads();
    t[4] = clock64();
    if (warp == 0) pk::warp_potrf32_s<pk::kDS>(S, ds, cbar, lane);
    __syncthreads();
    t[5] = clock64();
  }
  if (tid == 0) {
    g_probe[0] = t[1] - t[0];
    g_probe[1] = t[3] - t[2];
    g_probe[2] = t[5] - t[4];
  }
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
  const int smem = (64 * pk::kDS + 33 * 40) * 8;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 288, smem>>>(dA);
  cudaDeviceSynchronize();
  long long r[16];
  cudaMemcpyFromSymbol(r, g_probe, sizeof(r));
  printf("warp_diag32 alone %lld cycles, diag32 + tall32s %lld, old warp_potrf32 %lld (%s)\n", r[0], r[1], r[2],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
