// Two int8 (Ozaki) SYRK updates on concurrent streams vs the DMMA SYRK: locate wrong tiles.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "../paper_1805_00569_b200/csrc/kernels.cu"
#include "../paper_1805_00569_b200/csrc/ozaki_syrk.cuh"
using namespace pk;
static bool tmap_u8(CUtensorMap* m, const void* base, int64_t R, int64_t K, int box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)R, 8};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)(K * R)};
  cuuint32_t box[3] = {32u, (cuuint32_t)box_rows, 8u};
  cuuint32_t es[3] = {1u, 1u, 1u};
  return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
int main(int argc, char** argv) {
  const int NS = argc > 1 ? atoi(argv[1]) : 2;   // concurrent streams
  const int mp = argc > 2 ? atoi(argv[2]) : 4096;
  const int K = 512, row0 = K, R = mp - row0, T = R / 128;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<double> A((size_t)mp * mp);
  for (auto& v : A) v = nd(rng) * 0.3;
  cudaFuncSetAttribute(ozaki_syrk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kOzSmem);
  cudaFuncSetAttribute(dsyrk_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSyrkSmem);
  // reference (DMMA, serial)
  double* dR; cudaMalloc(&dR, A.size() * 8);
  cudaMemcpy(dR, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  CUtensorMap tR; make_tmap(&tR, dR, mp, mp, mp);
  SyrkParams u{}; u.row0 = row0; u.k0 = 0; u.ktiles = K / 16; u.T = T;
  dsyrk_persistent_kernel<<<T * (T + 1) / 2, kSyrkThreads, kSyrkSmem>>>(tR, u);
  cudaDeviceSynchronize();
  std::vector<double> ref(A.size());
  cudaMemcpy(ref.data(), dR, A.size() * 8, cudaMemcpyDeviceToHost);
  std::vector<double*> dA(NS); std::vector<int8_t*> sl(NS); std::vector<int*> ex(NS);
  std::vector<cudaStream_t> st(NS);
  std::vector<CUtensorMap> tA(NS), ta(NS), tb(NS);
  for (int i = 0; i < NS; ++i) {
    cudaMalloc(&dA[i], A.size() * 8); cudaMalloc(&sl[i], (size_t)8 * R * K); cudaMalloc(&ex[i], R * 4);
    cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
    make_tmap(&tA[i], dA[i], mp, mp, mp);
    tmap_u8(&ta[i], sl[i], R, K, 128); tmap_u8(&tb[i], sl[i], R, K, 64);
  }
  // optional background: NB streams each factorising an SPD matrix with the DMMA path
  const int NB = argc > 3 ? atoi(argv[3]) : 0;
  const int mb = argc > 4 ? atoi(argv[4]) : 4096;
  std::vector<double*> bK(NB), bA(NB), bL(NB); std::vector<int*> bst(NB);
  std::vector<CUtensorMap> btA(NB), btL(NB); std::vector<cudaStream_t> bs(NB);
  std::vector<double> spd((size_t)mb * mb);
  for (int i = 0; i < mb; ++i) for (int j = 0; j < mb; ++j) spd[(size_t)i * mb + j] = std::exp(-std::fabs(i - j) * 0.01) + (i == j ? 1.0 : 0.0);
  for (int i = 0; i < NB; ++i) {
    cudaMalloc(&bK[i], spd.size() * 8); cudaMalloc(&bA[i], spd.size() * 8); cudaMalloc(&bL[i], (size_t)mb * 128 * 8);
    cudaMemset(bL[i], 0, (size_t)mb * 128 * 8); cudaMalloc(&bst[i], 64); cudaMemset(bst[i], 0, 64);
    cudaMemcpy(bK[i], spd.data(), spd.size() * 8, cudaMemcpyHostToDevice);
    make_tmap(&btA[i], bA[i], mb, mb, mb); make_tmap(&btL[i], bL[i], mb, 128, 128);
    cudaStreamCreateWithFlags(&bs[i], cudaStreamNonBlocking);
  }
  Counter cnt;
  for (int rep = 0; rep < 3; ++rep) {
    for (int i = 0; i < NB; ++i)
      for (int r = 0; r < 4; ++r) {
        cudaMemcpyAsync(bA[i], bK[i], spd.size() * 8, cudaMemcpyDeviceToDevice, bs[i]);
        launch_potrf(bA[i], btA[i], btL[i], bL[i], mb, mb, bst[i], bs[i], cnt);
      }
    for (int i = 0; i < NS; ++i) cudaMemcpy(dA[i], A.data(), A.size() * 8, cudaMemcpyHostToDevice);
    cudaDeviceSynchronize();
    for (int i = 0; i < NS; ++i) {
      OzParams op{}; op.row0 = row0; op.R = R; op.ksteps = K / 32; op.exps = ex[i];
      ozaki_slice_kernel<<<(R * 32 + 255) / 256, 256, 0, st[i]>>>(dA[i], mp, row0, 0, R, K, sl[i], ex[i], nullptr, R);
      ozaki_syrk_kernel<<<T * (T + 1), kOzThreads, kOzSmem, st[i]>>>(ta[i], tb[i], tA[i], op);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    for (int i = 0; i < NS; ++i) {
      std::vector<double> got(A.size());
      cudaMemcpy(got.data(), dA[i], A.size() * 8, cudaMemcpyDeviceToHost);
      int bad = 0; int first_I = -1, first_J = -1; double worst = 0;
      for (int ti = 0; ti < T; ++ti)
        for (int tj = 0; tj <= 2 * ti + 1; ++tj) {
          double w = 0;
          for (int r = 0; r < 128; ++r)
            for (int c = 0; c < 64; ++c) {
              const size_t idx = (size_t)(row0 + ti * 128 + r) * mp + row0 + tj * 64 + c;
              w = std::max(w, std::fabs(got[idx] - ref[idx]));
            }
          if (w > 1e-10) { if (bad == 0) { first_I = ti; first_J = tj; } ++bad; }
          worst = std::max(worst, w);
        }
      printf("rep %d stream %d: bad tiles %d of %d, first (%d,%d), worst %.3e\n", rep, i, bad, T * (T + 1), first_I, first_J, worst);
    }
  }
  return 0;
}
