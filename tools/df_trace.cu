// Timeline of the dataflow Cholesky (potrf_df.cuh, PKRR_DF_TRACE): chain phase times per
// step and the worker tasks on the chain's critical path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/df_trace tools/df_trace.cu -lcuda
//   ./tools/df_trace [m] [dump.txt]
#define PKRR_DF_TRACE 1
#include "../paper_1805_00569_b200/csrc/kernels.cu"
#include <algorithm>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 4096;
  const int mp = (m + 127) / 128 * 128;
  std::vector<double> X(static_cast<size_t>(mp) * 20);
  srand(1);
  for (auto& v : X) v = (rand() / (double)RAND_MAX - 0.5) * 3.0;
  std::vector<double> A(static_cast<size_t>(mp) * mp);
  for (int i = 0; i < mp; ++i)
    for (int j = 0; j < mp; ++j) {
      double d2 = 0;
      for (int t = 0; t < 20; ++t) {
        const double df = X[i * 20 + t] - X[j * 20 + t];
        d2 += df * df;
      }
      A[static_cast<size_t>(i) * mp + j] = exp(-d2 / 18.0) + (i == j ? 1e-3 * mp : 0.0);
    }
  double *dA, *dL, *y, *w, *z;
  int* st;
  cudaMalloc(&dA, sizeof(double) * mp * mp);
  cudaMalloc(&dL, sizeof(double) * mp * 128);
  cudaMalloc(&y, sizeof(double) * mp);
  cudaMalloc(&w, sizeof(double) * mp);
  cudaMalloc(&z, sizeof(double) * mp);
  cudaMalloc(&st, 8);
  cudaMemset(y, 0, sizeof(double) * mp);
  CUtensorMap tmA, tmL;
  pk::make_tmap(&tmA, dA, mp, mp, mp);
  pk::make_tmap(&tmL, dL, mp, 128, 128);
  pk::Counter c;
  pk::FwdSolve fs{y, w, z};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemcpy(dA, A.data(), sizeof(double) * mp * mp, cudaMemcpyHostToDevice);
    cudaMemset(st, 0, 8);
    cudaEventRecord(e0);
    pk::launch_potrf(dA, tmA, tmL, dL, mp, m, st, 0, c, nullptr, nullptr, nullptr, true, &fs);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("m %d: %.3f ms (%s)\n", m, ms, cudaGetErrorString(cudaGetLastError()));
  const int nt = mp / 64;
  std::vector<int4> tasks = pk::df_build_tasks(nt, false);
  static unsigned long long ch[256][12];
  static unsigned long long tk[65536][4];
  cudaMemcpyFromSymbol(ch, pk::g_df_chain, sizeof(ch));
  for (int k = 0; k < 256; ++k)
    for (int i = 0; i < 12; ++i) if (i != 9 && i != 11) ch[k][i] = (unsigned long long)(ch[k][i] / 1.965);  // cycles -> ns
  cudaMemcpyFromSymbol(tk, pk::g_df_task, sizeof(tk));
  const unsigned long long t0 = ch[0][0];
  const char* names[] = {"start", "T ready", "diag0 done", "sub0", "syrk", "sub1", "inv", "fwd", "publish",
                         "prep wait", "prep done"};
  double avg[12] = {};
  int cnt = 0;
  for (int k = 1; k < nt - 1; ++k, ++cnt)
    for (int i = 1; i <= 10; ++i) avg[i] += (double)(ch[k][i] - ch[k][0]) / 1e3;
  printf("chain phases (us after step start, mean over steps 1..nt-2):");
  for (int i = 1; i <= 10; ++i) printf("  %s %.2f", names[i], avg[i] / cnt);
  printf("\nstep length (us):");
  for (int k = 0; k + 1 < nt; ++k) printf(" %.1f", (ch[k + 1][0] - ch[k][0]) / 1e3);
  printf("\n");
  // critical worker tasks per step k (globaltimer us after the step's start): TRSM(k+1, k-1)
  // -> UPD(k+1, k, {k-1}) -> T(k), UPD(k+1, k+1, {k-1}) -> D(k+1)
  static unsigned long long wt0[256][8][8];
  cudaMemcpyFromSymbol(wt0, pk::g_df_warp, sizeof(wt0));
  for (int k : {4, 12, 14, 16, 20, 24, 40, 41}) {
    if (k >= nt - 1) continue;
    const long long s0 = (long long)ch[k][11];
    printf("step %d (len %.1f): publish(k-1) %.1f, L(k,k-1) out %.1f, publish(k) %.1f", k,
           ((long long)ch[k + 1][11] - s0) / 1e3, ((long long)ch[k - 1][9] - s0) / 1e3,
           ((long long)wt0[k][4][0] - s0) / 1e3, ((long long)ch[k][9] - s0) / 1e3);
    for (size_t t = 0; t < tasks.size(); ++t) {
      const int4 q = tasks[t];
      const int a = q.w & 0xffff, b = q.w >> 16;
      if ((q.x == pk::DF_TRSM && q.y == k + 1 && q.z == k - 1) ||
          (q.x == pk::DF_UPD && q.y == k + 1 && q.z == k && b == k) ||
          (q.x == pk::DF_UPD && q.y == k + 1 && q.z == k + 1 && b == k))
        printf("  [%s %d,%d %d-%d #%zu: claim %.1f ready %.1f done %.1f cta %llu]", q.x == pk::DF_TRSM ? "TRSM" : "UPD",
               q.y, q.z, a, b, t, ((long long)tk[t][0] - s0) / 1e3, ((long long)tk[t][1] - s0) / 1e3,
               ((long long)tk[t][2] - s0) / 1e3, tk[t][3]);
    }
    printf("\n");
  }
  // worker utilisation: busy time (ready -> done) / (workers * span)
  unsigned long long tend = 0;
  double busy = 0;
  double wait = 0;
  for (size_t t = 0; t < tasks.size(); ++t) {
    tend = std::max(tend, tk[t][2]);
    busy += (double)(tk[t][2] - tk[t][1]);
    wait += (double)(tk[t][1] - tk[t][0]);
  }
  printf("tasks %zu, span %.1f us, worker busy %.1f%%, mean dep wait %.2f us, mean task %.2f us\n", tasks.size(),
         (tend - t0) / 1e3, 100.0 * busy / (147.0 * (tend - t0)), wait / tasks.size() / 1e3,
         busy / tasks.size() / 1e3);
  static unsigned long long wt[256][8][8];
  cudaMemcpyFromSymbol(wt, pk::g_df_warp, sizeof(wt));
  for (int k = 0; k < 256; ++k)
    for (int w = 0; w < 8; ++w)
      for (int i = 0; i < 8; ++i) wt[k][w][i] = (unsigned long long)(wt[k][w][i] / 1.965);
  for (int k : {8, 40, 41}) {
    const long long c0 = (long long)ch[k][0];
    printf("step %d chain marks (us):", k);
    for (int i = 1; i <= 10; ++i) printf(" m%d %.2f", i, ((long long)ch[k][i] - c0) / 1e3);
    printf("  next-start %.2f\n", ((long long)ch[k + 1][0] - c0) / 1e3);
    for (int w = 0; w < 8; ++w) {
      if (w == 4) continue;
      printf("   w%d: A-start %.2f A-work %.2f pre-csync1 %.2f B-work %.2f C-work %.2f D-work %.2f zpub %.2f Trows %.2f\n", w,
             ((long long)wt[k][w][0] - c0) / 1e3, ((long long)wt[k][w][1] - c0) / 1e3,
             ((long long)wt[k][w][5] - c0) / 1e3, ((long long)wt[k][w][2] - c0) / 1e3,
             ((long long)wt[k][w][3] - c0) / 1e3, ((long long)wt[k][w][4] - c0) / 1e3,
             ((long long)wt[k][w][6] - c0) / 1e3, ((long long)wt[k][w][7] - c0) / 1e3);
    }
  }
  if (argc > 2) {
    FILE* f = fopen(argv[2], "w");
    for (size_t t = 0; t < tasks.size(); ++t) {
      const int4 q = tasks[t];
      fprintf(f, "%zu %d %d %d %d %d %lld %lld %lld %llu\n", t, q.x, q.y, q.z, q.w & 0xffff, q.w >> 16,
              (long long)tk[t][0] - (long long)t0, (long long)tk[t][1] - (long long)t0,
              (long long)tk[t][2] - (long long)t0, tk[t][3]);
    }
    for (int k = 0; k < nt; ++k) {
      fprintf(f, "C %d", k);
      for (int i = 0; i <= 10; ++i) fprintf(f, " %lld", (long long)ch[k][i] - (long long)t0);
      fprintf(f, "\n");
    }
    fclose(f);
  }
  return 0;
}
