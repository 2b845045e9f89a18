// Determinism probe for the whole blocked Cholesky (launch_potrf): NS streams each
// factorise private copies of the same SPD matrix; every factor must equal the serial one.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "../paper_1805_00569_b200/csrc/kernels.cu"
using namespace pk;
int main(int argc, char** argv) {
  const int NS = argc > 1 ? atoi(argv[1]) : 8;
  const int mp = argc > 2 ? atoi(argv[2]) : 4096;
  const int reps = argc > 3 ? atoi(argv[3]) : 5;
  if (argc > 4) set_panel_group(atoi(argv[4]));
  const int oz = argc > 5 ? atoi(argv[5]) : 0;
  set_syrk_ozaki(oz);
  std::vector<double> K((size_t)mp * mp);
  std::mt19937_64 rng(5);
  std::uniform_real_distribution<double> ud(-1.0, 1.0);
  std::vector<double> x(mp * 3);
  for (auto& v : x) v = ud(rng);
  for (int i = 0; i < mp; ++i)
    for (int j = 0; j < mp; ++j) {
      double d2 = 0;
      for (int t = 0; t < 3; ++t) d2 += (x[i * 3 + t] - x[j * 3 + t]) * (x[i * 3 + t] - x[j * 3 + t]);
      K[(size_t)i * mp + j] = std::exp(-d2 / 0.5) + (i == j ? 1e-3 * mp : 0.0);
    }
  double* dK;
  cudaMalloc(&dK, K.size() * 8);
  cudaMemcpy(dK, K.data(), K.size() * 8, cudaMemcpyHostToDevice);
  struct Buf { double* A; double* L; int* st; int8_t* sl; int* ex; CUtensorMap tA, tL; };
  auto mk = [&]() {
    Buf b;
    cudaMalloc(&b.A, K.size() * 8);
    cudaMalloc(&b.L, (size_t)mp * kNB * 8);
    cudaMalloc(&b.st, 64);
    cudaMalloc(&b.sl, (size_t)2 * 8 * mp * 512);
    cudaMalloc(&b.ex, (size_t)2 * mp * 4);
    make_tmap(&b.tA, b.A, mp, mp, mp);
    make_tmap(&b.tL, b.L, mp, kNB, kNB);
    return b;
  };
  Counter c;
  Buf R = mk();
  cudaMemcpy(R.A, dK, K.size() * 8, cudaMemcpyDeviceToDevice);
  cudaMemset(R.L, 0, (size_t)mp * kNB * 8);
  cudaMemset(R.st, 0, 64);
  launch_potrf(R.A, R.tA, R.tL, R.L, mp, mp, R.st, 0, c, R.sl, R.ex);
  // oz == 2: odd streams run the DMMA path -> their reference is the DMMA factor
  std::vector<double> ref_dmma(K.size());
  if (oz == 2) {
    Buf R2 = mk();
    cudaMemcpy(R2.A, dK, K.size() * 8, cudaMemcpyDeviceToDevice);
    cudaMemset(R2.L, 0, (size_t)mp * kNB * 8);
    cudaMemset(R2.st, 0, 64);
    launch_potrf(R2.A, R2.tA, R2.tL, R2.L, mp, mp, R2.st, 0, c, nullptr, nullptr);
    cudaDeviceSynchronize();
    cudaMemcpy(ref_dmma.data(), R2.A, K.size() * 8, cudaMemcpyDeviceToHost);
  }
  cudaDeviceSynchronize();
  std::vector<double> ref(K.size()), got(K.size());
  cudaMemcpy(ref.data(), R.A, K.size() * 8, cudaMemcpyDeviceToHost);
  int st0[2];
  cudaMemcpy(st0, R.st, 8, cudaMemcpyDeviceToHost);
  printf("serial status %d %d\n", st0[0], st0[1]);
  std::vector<Buf> B(NS);
  std::vector<cudaStream_t> s(NS);
  for (int i = 0; i < NS; ++i) {
    B[i] = mk();
    cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking);
  }
  int wrong = 0, wrong_odd = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int i = 0; i < NS; ++i) {
      cudaMemcpyAsync(B[i].A, dK, K.size() * 8, cudaMemcpyDeviceToDevice, s[i]);
      cudaMemsetAsync(B[i].L, 0, (size_t)mp * kNB * 8, s[i]);
      cudaMemsetAsync(B[i].st, 0, 64, s[i]);
    }
    for (int i = 0; i < NS; ++i) launch_potrf(B[i].A, B[i].tA, B[i].tL, B[i].L, mp, mp,
                                             (oz == 2 && !(i & 1)) ? nullptr : B[i].st, s[i], c,
                                             (oz == 2 && (i & 1)) ? nullptr : B[i].sl, B[i].ex);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    for (int i = 0; i < NS; ++i) {
      cudaMemcpy(got.data(), B[i].A, K.size() * 8, cudaMemcpyDeviceToHost);
      long bad = 0, first = -1;
      for (int r = 0; r < mp; ++r)
        for (int cc = 0; cc <= r; ++cc) {
          const size_t xx = (size_t)r * mp + cc;
          const double want = (oz == 2 && (i & 1)) ? ref_dmma[xx] : ref[xx];
          if (got[xx] != want) { if (first < 0) first = xx; ++bad; }
        }
      if (bad) { ++wrong; if (i & 1) ++wrong_odd; printf("rep %d stream %d: %ld wrong (lower), first row %ld col %ld\n", rep, i, bad, first / mp, first % mp); }
    }
  }
  if (std::getenv("PKRR_SHADOW")) shadow_report();
  printf("NS=%d mp=%d reps=%d: %d wrong factors (%d on odd streams)\n", NS, mp, reps, wrong, wrong_odd);
  return 0;
}
