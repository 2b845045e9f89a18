// Phase timing of the Cholesky leaf kernel (clock64 stamps, PKRR_LEAF_TRACE).
#define PKRR_LEAF_TRACE 1
#include "../paper_1805_00569_b200/csrc/kernels.cu"
#include <vector>
#include <cstdlib>
int main() {
  const int m = 128;
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
  double *dA, *dL;
  int* st;
  cudaMalloc(&dA, m * m * 8);
  cudaMalloc(&dL, m * m * 8);
  cudaMalloc(&st, 8);
  cudaFuncSetAttribute(pk::potrf_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pk::kLeafSmem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(dA, A.data(), m * m * 8, cudaMemcpyHostToDevice);
    cudaMemset(st, 0, 8);
    pk::potrf_leaf_kernel<<<1, pk::kLeafThreads, pk::kLeafSmem>>>(dA, m, 0, dL, st, m, 1);
    cudaDeviceSynchronize();
  }
  long long tr[64];
  cudaMemcpyFromSymbol(tr, pk::g_leaf_trace, sizeof(tr));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  const char* names[] = {"issue", "load", "p0", "potrf0", "trtri0", "trsm0", "p1", "potrf1", "trtri1", "trsm1",
                         "p2", "potrf2", "trtri2", "trsm2", "p3", "potrf3", "trtri3", "trsm3"};
  for (int i = 1; i <= 24; ++i) printf("%2d %8lld\n", i, tr[i] - tr[i - 1]);
  printf("total %lld cycles\n", tr[24] - tr[0]);
  for (int pb = 0; pb < 4; ++pb) {
    printf("panel %d: diag warp %lld", pb, tr[40 + pb] - tr[2 + 5 * pb]);
    for (int w = 1; w < 4 - pb; ++w) printf("  tall warp %d %lld", w, tr[44 + 4 * pb + w] - tr[2 + 5 * pb]);
    printf("  all %lld\n", tr[3 + 5 * pb] - tr[2 + 5 * pb]);
  }
}
