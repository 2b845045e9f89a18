// Determinism probe for the in-place panel TRSM (dgemm_tn_kernel<64, G_STORE>):
// NS streams each run the same TRSM on private copies of the same input, repeatedly,
// optionally with other kernels alongside; every result must equal the serial one.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "../paper_1805_00569_b200/csrc/kernels.cu"
__global__ void noise_kernel(const double* __restrict__ A, int64_t lda, int R, int K, int8_t* out, int* e) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= R) return;
  const double* row = A + static_cast<int64_t>(warp) * lda;
  double mx = 0.0;
  for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(row[k]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int ex = mx > 0.0 ? ilogb(mx) + 2 : 0;
  if (lane == 0) e[warp] = ex;
  for (int k = lane; k < K; k += 32) {
    double x = ldexp(row[k], -ex);
    for (int s = 0; s < 8; ++s) {
      const double t = x * 128.0;
      const double d = rint(t);
      out[(static_cast<int64_t>(s) * R + warp) * K + k] = static_cast<int8_t>(d);
      x = t - d;
    }
  }
}
using namespace pk;
int main(int argc, char** argv) {
  const int NS = argc > 1 ? atoi(argv[1]) : 8;
  const int mp = argc > 2 ? atoi(argv[2]) : 4096;
  const int reps = argc > 3 ? atoi(argv[3]) : 20;
  const int kb = argc > 4 ? atoi(argv[4]) : 0;
  const int nb = mp / kNB, rem = nb - 1 - kb;
  std::mt19937_64 rng(11);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<double> A((size_t)mp * mp), L((size_t)mp * kNB, 0.0);
  for (auto& v : A) v = nd(rng);
  for (int r = 0; r < mp; ++r)
    for (int c = 0; c <= (r % kNB); ++c) L[(size_t)r * kNB + c] = nd(rng);
  double *dA0, *dL;
  cudaMalloc(&dA0, A.size() * 8);
  cudaMalloc(&dL, L.size() * 8);
  cudaMemcpy(dA0, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dL, L.data(), L.size() * 8, cudaMemcpyHostToDevice);
  CUtensorMap tL;
  make_tmap(&tL, dL, mp, kNB, kNB);
  auto trsm = [&](double* a, const CUtensorMap& ta, cudaStream_t s) {
    GemmParams t{};
    t.a_row0 = (kb + 1) * kNB;
    t.a_k0 = kb * kNB;
    t.b_row0 = kb * kNB;
    t.b_k0 = 0;
    t.ktiles = kNB / kBK;
    t.C = a;
    t.ldc = mp;
    t.c_row0 = (kb + 1) * kNB;
    t.c_col0 = kb * kNB;
    t.tiles_m = rem * 2;
    t.tiles_n = 1;
    Counter c;
    gemm_launch<64, G_STORE>(ta, tL, t, rem * 2, s, c);
  };
  // serial reference
  double* dR;
  cudaMalloc(&dR, A.size() * 8);
  cudaMemcpy(dR, dA0, A.size() * 8, cudaMemcpyDeviceToDevice);
  CUtensorMap tR;
  make_tmap(&tR, dR, mp, mp, mp);
  trsm(dR, tR, 0);
  cudaDeviceSynchronize();
  std::vector<double> ref(A.size());
  cudaMemcpy(ref.data(), dR, A.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<double*> dA(NS);
  std::vector<CUtensorMap> tA(NS);
  std::vector<cudaStream_t> st(NS);
  for (int i = 0; i < NS; ++i) {
    cudaMalloc(&dA[i], A.size() * 8);
    make_tmap(&tA[i], dA[i], mp, mp, mp);
    cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  }
  const int NN = argc > 5 ? atoi(argv[5]) : 0;  // noise streams
  std::vector<cudaStream_t> ns(NN);
  int8_t* nbuf; int* nex;
  cudaMalloc(&nbuf, (size_t)8 * mp * 512);
  cudaMalloc(&nex, mp * 4);
  for (int i = 0; i < NN; ++i) cudaStreamCreateWithFlags(&ns[i], cudaStreamNonBlocking);
  int bad_total = 0;
  std::vector<double> got(A.size());
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = 0; i < NS; ++i) cudaMemcpyAsync(dA[i], dA0, A.size() * 8, cudaMemcpyDeviceToDevice, st[i]);
    cudaDeviceSynchronize();
    for (int j = 0; j < NN; ++j)
      for (int r = 0; r < 20; ++r) noise_kernel<<<mp / 8, 256, 0, ns[j]>>>(dA0, mp, mp, 512, nbuf, nex);
    for (int t = 0; t < 8; ++t)
      for (int i = 0; i < NS; ++i) {
        if (t) cudaMemcpyAsync(dA[i], dA0, A.size() * 8, cudaMemcpyDeviceToDevice, st[i]);
        trsm(dA[i], tA[i], st[i]);
      }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("err %s\n", cudaGetErrorString(e));
      return 1;
    }
    for (int i = 0; i < NS; ++i) {
      cudaMemcpy(got.data(), dA[i], A.size() * 8, cudaMemcpyDeviceToHost);
      long bad = 0, rmin = 1 << 30, rmax = -1, cmin = 1 << 30, cmax = -1;
      for (size_t x = 0; x < got.size(); ++x)
        if (got[x] != ref[x]) {
          ++bad;
          const long r = x / mp, c = x % mp;
          rmin = std::min(rmin, r); rmax = std::max(rmax, r);
          cmin = std::min(cmin, c); cmax = std::max(cmax, c);
        }
      if (bad) {
        ++bad_total;
        printf("rep %d stream %d: %ld wrong, rows [%ld,%ld] cols [%ld,%ld]\n", rep, i, bad, rmin, rmax, cmin, cmax);
      }
    }
  }
  printf("NS=%d mp=%d kb=%d reps=%d: %d wrong results\n", NS, mp, kb, reps, bad_total);
  return 0;
}
