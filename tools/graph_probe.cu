// Is the m x m factorization (C0: m = 4096) launch-gap bound?  Times launch_potrf as
// direct launches vs the same sequence captured into a CUDA graph and replayed.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_1805_00569_b200/csrc/kernels.cu"
using namespace pk;
int main(int argc, char** argv) {
  const int mp = argc > 1 ? atoi(argv[1]) : 4096;
  const bool look = argc > 2 ? atoi(argv[2]) : 1;
  std::vector<double> K((size_t)mp * mp);
  for (int i = 0; i < mp; ++i)
    for (int j = 0; j < mp; ++j) K[(size_t)i * mp + j] = std::exp(-std::fabs(i - j) * 0.01) + (i == j ? 0.5 * mp * 1e-3 : 0.0);
  double *dK, *A, *L;
  int* st;
  cudaMalloc(&dK, K.size() * 8);
  cudaMalloc(&A, K.size() * 8);
  cudaMalloc(&L, (size_t)mp * 128 * 8);
  cudaMalloc(&st, 64);
  cudaMemcpy(dK, K.data(), K.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(L, 0, (size_t)mp * 128 * 8);
  cudaMemset(st, 0, 64);
  CUtensorMap tA, tL;
  make_tmap(&tA, A, mp, mp, mp);
  make_tmap(&tL, L, mp, 128, 128);
  int lo, hi;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStream_t s, s2;
  cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi);
  cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, lo);
  Counter c;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&] {
    cudaMemcpyAsync(A, dK, K.size() * 8, cudaMemcpyDeviceToDevice, s);
    launch_potrf(A, tA, tL, L, mp, mp, st, s, c, nullptr, nullptr, look ? s2 : nullptr);
  };
  for (int w = 0; w < 3; ++w) run();
  cudaStreamSynchronize(s);
  float ms = 0;
  cudaEventRecord(a, s);
  for (int w = 0; w < 10; ++w) run();
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  const long long launches = c.launches;
  printf("m=%d lookahead=%d direct: %.3f ms per factorization (incl. %.3f ms copy)\n", mp, (int)look, ms / 10,
         K.size() * 8 * 2 / 5.5e9);
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  run();
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ge;
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
    printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 1;
  }
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  size_t nodes = 0;
  cudaGraphGetNodes(g, nullptr, &nodes);
  printf("m=%d lookahead=%d graph : %.3f ms per factorization (%zu nodes, %lld launches per call)\n", mp, (int)look,
         ms / 10, nodes, launches / 14);
  return 0;
}
