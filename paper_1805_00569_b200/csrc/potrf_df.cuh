// potrf_df.cuh -- dataflow Cholesky for a system factorised ALONE (latency mode,
// mp < 8192: BASELINE configs[0], pkrrgpu_cholesky / train_krr on one system).
//
// The stream-ordered blocked path (launch_potrf) runs one 128-column panel step as
// leaf -> TRSM -> next-column update kernels; for a lone 4096-row system that chain
// (≈ 57 µs per panel, the leaf alone 40 µs on a cold SM) and the K = 128 trailing
// updates' wave tails bound the factorization at ≈ 2.1 ms (profiles/).
// Here ONE persistent cooperative kernel does the whole factorization:
//
//  * the chain CTA (the first CTA to start) walks the 64-column panels k = 0..nt-1
//    without ever leaving the SM: factor the diagonal tile (two 32-column warp
//    panels, the reference's column loop solver.cpp:18-33), factor the tile below it
//    (k+1, k) along with it one column behind (the panel TRSM for the next tile row,
//    by substitution), invert L_kk (64 x 64), advance the forward substitution
//    z_k = inv(L_kk) (y_k - sum_p L(k,p) z_p), publish, then apply panel k to the next
//    diagonal tile in shared memory;
//  * every other CTA is a worker pulling tile tasks from a static list: TRSM(i, k)
//    (L(i,k) = A(i,k) inv(L_kk)^T as a DMMA GEMM, plus its L(i,k) z_k share of the
//    forward substitution), UPD(i, j, [a, b)) (A(i,j) -= sum_{q in [a,b)} L(i,q) L(j,q)^T,
//    far panels batched 8 at a time -- K = 512 -- the last two singly, so the tiles
//    near the diagonal are ready a step after their panel), INV(b) (the 128 x 128
//    diagonal-block inverse the backward solve uses).  Operands and C tiles move by
//    TMA into a ring (producer warp; TRSMs and single updates stream each operand as soon
//    as its own producer is done), 4 DMMA warps (32 x 32 each) compute, a publisher warp
//    issues the tasks' release stores;
//  * dependencies are per-tile counters in global memory (release / acquire):
//    applied[i][j] = panels applied to tile (i,j), lrow[i] = L tiles of row i done,
//    chain = panels finished.  The task list is a topological order with the chain
//    steps as virtual nodes (a task that waits on chain step k comes after every task
//    chain step k waits on), claimed through one atomic ticket: with all CTAs
//    co-resident (cooperative launch) the schedule cannot deadlock.
//
// Every tile receives its panels in a fixed order with fixed arithmetic, so the
// factor is bitwise reproducible run to run; it differs from the 128-blocked path
// only by summation order (parity vs the oracle: tests/test_gpu_parity.py, C0 golden).
#pragma once

namespace pk {

constexpr int kDfT = 64;                  // tile
constexpr int kDfThreads = 8 * 32;        // workers: 4 DMMA warps + TMA producer warp + publisher warp (+ 2 idle);
                                          // 2 warps per scheduler partition -> up to 255 registers
constexpr int kDfStages = 8;
constexpr int kDfStage = 2 * kDfT * kBK * 8;  // A box + B box (64 rows x 16) = 16 KB
constexpr int kDfCbuf = kDfT * kDfT * 8;      // one C tile (4 swizzled 64x16 boxes) = 32 KB
constexpr int kDS = 68;                       // chain smem row stride (== 4 mod 16: conflict-free fragments)
constexpr int kDfSingles = 2;                 // trailing panels applied one at a time per tile
constexpr int kDfBatch = 8;                   // far panels per update task (K = 512)
constexpr int kDfWorkerSmem = kDfStages * kDfStage + 2 * kDfCbuf + 4 * 64 * 8 + 32 * 8 + 64;
constexpr int kDfChainSmem = (5 * 64 * kDS + 32 * 32 + 8 * 64) * 8 + 8 * 8 + 64;
constexpr int kDfSmem = (kDfWorkerSmem > kDfChainSmem ? kDfWorkerSmem : kDfChainSmem) + 1024;

#ifdef PKRR_DF_TRACE
// debug timeline (tools/df_trace.cu): chain phase stamps per step, per-task claim /
// dependencies-met / done stamps (globaltimer ns)
__device__ unsigned long long g_df_chain[256][12];
__device__ unsigned long long g_df_task[65536][4];
__device__ unsigned long long g_df_warp[256][8][8];
__device__ __forceinline__ unsigned long long df_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
// chain stamps: the SM's cycle counter (consistent across the chain's warps; globaltimer
// is not, below ~1 us), converted at 1.965 GHz by the tool
__device__ __forceinline__ unsigned long long df_clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  return t;
}
#define DF_CHAIN_MARK(k, i) \
  if (threadIdx.x == 0) g_df_chain[k][i] = df_clk();
#define DF_TASK_MARK(t, i, v) g_df_task[t][i] = (v);
#else
#define DF_CHAIN_MARK(k, i)
#define DF_TASK_MARK(t, i, v)
#endif

enum DfType { DF_TRSM = 0, DF_UPD = 1, DF_INV = 2, DF_END = 3, DF_GRAM = 4 };
// flag words (ints) at the head of the workspace
enum DfFlag { F_TICKET = 0, F_ROLE = 1, F_CHAIN = 2, F_HEAD = 8 };

struct DfParams {
  double* A;
  int64_t lda;
  int nt;                // tiles of 64
  double* inv64;         // [nt][64][64] inverses of the 64-row diagonal blocks
  double* P;             // [nt][nt][64] forward-substitution shares L(i,k) z_k
  double* Linv;          // [mp][128] inverses of the 128-row diagonal blocks (backward solve)
  const double* y;       // forward substitution right-hand side (null: factor only)
  double* z;
  int* status;           // [2] abort flag, first failing column
  int* flags;            // F_HEAD ints, applied[nt*nt], lrow[nt]
  const int4* tasks;     // {type, i, j, a | b << 16}
  int ntasks;
  // fused kernel-matrix build (gram != 0): GRAM(i, j) tasks form tile (i, j) of
  // K = exp(-|x_i - x_j|^2 / ((2 s) s)) (kernel.cpp:52-56) from the padded rows X (tmX,
  // xk 16-column chunks) and their norms, write it to K and K + shift I to A
  int gram;
  int xk;
  int m_valid;
  const double* xnorm;
  double* K;
  double neg_inv_denom;
  double shift;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// async-proxy reads (TMA / bulk copies) of global data published by generic stores of
// other CTAs, after the acquire that observed the publication
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// spin until *flag >= target; false if the factorization was abandoned (NPD).  A wait
// that exceeds ~2^33 cycles is a scheduling bug: trap (a loud launch failure) instead of
// hanging the GPU.
__device__ __noinline__ bool df_wait_ge(const int* flag, int target, const int* abort_flag) {
  // relaxed polling + one acquire load on success: an ld.acquire per poll invalidates
  // the SM's L1 every iteration
  const volatile int* f = flag;
  if (*f < target) {
    const long long t0 = clock64();
    while (*f < target) {
      if (*reinterpret_cast<const volatile int*>(abort_flag)) return false;
      if (clock64() - t0 > (1ll << 33)) __trap();
      __nanosleep(32);
    }
  }
  // one acquire load (orders what follows) -- not a fence.acq_rel, which would also wait
  // for this thread's outstanding bulk copies (microseconds under the workers' traffic)
  (void)ld_acquire_gpu(flag);
  return true;
}

// ---------------------------------------------------------------------------
// worker: TMA producer warp + 4 DMMA warps (2 x 2 grid, 32 x 32 per warp) + publisher warp
// ---------------------------------------------------------------------------
__device__ __forceinline__ void df_worker(const CUtensorMap* tmA, const CUtensorMap* tmI, const CUtensorMap* tmX,
                                          const DfParams& p,
                                          unsigned char* smem) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt = p.nt;
  unsigned char* ring = smem;
  unsigned char* cbuf = smem + kDfStages * kDfStage;
  double* red = reinterpret_cast<double*>(cbuf + 2 * kDfCbuf);  // [4][64]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 4 * 64);
  uint64_t* empty = full + kDfStages;
  uint64_t* tfull = empty + kDfStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* cfull = tempty + 2;
  uint64_t* cempty = cfull + 2;
  int4* tslot = reinterpret_cast<int4*>(cempty + 2);
#ifdef PKRR_DF_TRACE
  __shared__ int tticket[2];
  __shared__ int pticket[2];
#endif
  __shared__ uint64_t pubfull[2], pubempty[2];
  __shared__ int4 ptask[2];
  int* applied = p.flags + F_HEAD;
  int* lrow = applied + nt * nt;
  if (tid == 0) {
    for (int s = 0; s < kDfStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], 4);
      mbar_init(&pubfull[s], 4);
      mbar_init(&pubempty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp >= 6) return;
  if (warp == 5) {
    // ---------------- publisher: the tasks' release stores ----------------
    // st.release.gpu waits (MEMBAR.ALL.GPU, ~0.7 us under the workers' traffic) for the
    // CTA's stores to be visible; on a DMMA warp that wait was added to every task (the
    // other three warps met it again at the next task's barrier).  The four DMMA warps
    // arrive on pubfull[slot] when their stores are issued; this thread publishes.
    if (lane != 0) return;
    for (int it = 0;; ++it) {
      const int slot = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      mbar_wait(&pubfull[slot], ph);
      const int4 task = ptask[slot];
      if (task.x == DF_END) return;
      const int ti = task.y, tj = task.z, tb = task.w >> 16;
      if (task.x == DF_UPD) st_release_gpu(applied + ti * nt + tj, tb);
      else if (task.x == DF_TRSM) st_release_gpu(lrow + ti, tj + 1);
      else if (task.x == DF_GRAM) st_release_gpu(applied + ti * nt + tj, 0);
#ifdef PKRR_DF_TRACE
      DF_TASK_MARK(pticket[slot], 2, df_now());
#endif
      mbar_arrive(&pubempty[slot]);
    }
  }
  if (warp == 4) {
    // ---------------- producer: claim, wait for dependencies, stream operands ----------------
    if (lane != 0) return;
    prefetch_tmap(tmA);
    prefetch_tmap(tmI);
    if (p.gram) prefetch_tmap(tmX);
    int kt = 0;
    for (int it = 0;; ++it) {
      const int t = atomicAdd(p.flags + F_TICKET, 1);
      int4 task = t < p.ntasks ? p.tasks[t] : make_int4(DF_END, 0, 0, 0);
#ifdef PKRR_DF_TRACE
      if (t < p.ntasks) DF_TASK_MARK(t, 0, df_now());
#endif
      const int ti = task.y, tj = task.z, ta = task.w & 0xffff, tb = task.w >> 16;
      // TRSMs and single updates (K = 64, the tasks the chain's next steps wait for) stream
      // each operand as soon as ITS producer is done instead of after the last dependency:
      // the C tile / A rows are in flight while the task still waits for the chain's
      // publication, and only the B rows' TMA latency follows it
      const bool split = task.x == DF_TRSM || (task.x == DF_UPD && tb - ta == 1);
      bool ok = true;
      if (split) {
        ok = df_wait_ge(applied + ti * nt + tj, task.x == DF_TRSM ? tj : ta, p.status);
      } else if (task.x == DF_UPD) {
        ok = df_wait_ge(applied + ti * nt + tj, ta, p.status) && df_wait_ge(lrow + ti, tb, p.status) &&
             df_wait_ge(lrow + tj, tb, p.status);
      } else if (task.x == DF_INV) {
        ok = df_wait_ge(p.flags + F_CHAIN, 2 * ti + 2, p.status);
      }
      if (!ok) task.x = DF_END;
#ifdef PKRR_DF_TRACE
      if (t < p.ntasks) {
        if (!split) DF_TASK_MARK(t, 1, df_now());
        DF_TASK_MARK(t, 3, blockIdx.x);
      }
      tticket[it & 1] = t;
#endif
      fence_proxy_async_global();
      const int slot = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      mbar_wait(&tempty[slot], ph ^ 1);
      tslot[slot] = task;
      mbar_arrive(&tfull[slot]);
      if (task.x == DF_END) return;
      mbar_wait(&cempty[slot], ph ^ 1);
      if (task.x == DF_UPD) {
        mbar_arrive_expect_tx(&cfull[slot], kDfCbuf);
#pragma unroll
        for (int h = 0; h < 4; ++h) tma_load_2d(cbuf + slot * kDfCbuf + h * 8192, tmA, tj * kDfT + 16 * h, ti * kDfT,
                                                &cfull[slot]);
      } else {
        mbar_arrive(&cfull[slot]);
      }
      if (split) {
        // (an abandoned factorization -- a wait returning false -- still issues every load:
        // the consumers are already waiting on these stages; the next claim ends the worker)
        const bool trsm = task.x == DF_TRSM;
        if (!trsm) {
          (void)df_wait_ge(lrow + ti, tb, p.status);
          fence_proxy_async_global();
        }
        for (int c = 0; c < 4; ++c) {
          const int s = (kt + c) % kDfStages;
          mbar_wait(&empty[s], (((kt + c) / kDfStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], kDfStage);
          tma_load_2d(ring + s * kDfStage, tmA, (trsm ? tj : ta) * kDfT + 16 * c, ti * kDfT, &full[s]);
        }
        (void)df_wait_ge(trsm ? p.flags + F_CHAIN : lrow + tj, trsm ? tj + 1 : tb, p.status);
        fence_proxy_async_global();
#ifdef PKRR_DF_TRACE
        DF_TASK_MARK(t, 1, df_now());
#endif
        for (int c = 0; c < 4; ++c) {
          unsigned char* sb = ring + ((kt + c) % kDfStages) * kDfStage + 8192;
          if (trsm) tma_load_2d(sb, tmI, 16 * c, tj * kDfT, &full[(kt + c) % kDfStages]);
          else tma_load_2d(sb, tmA, ta * kDfT + 16 * c, tj * kDfT, &full[(kt + c) % kDfStages]);
        }
        kt += 4;
        continue;
      }
      const int nk = task.x == DF_UPD ? 4 * (tb - ta) : (task.x == DF_GRAM ? p.xk : 0);
      for (int c = 0; c < nk; ++c, ++kt) {
        const int s = kt % kDfStages;
        const uint32_t sp = (kt / kDfStages) & 1;
        mbar_wait(&empty[s], sp ^ 1);
        mbar_arrive_expect_tx(&full[s], kDfStage);
        unsigned char* sa = ring + s * kDfStage;
        if (task.x == DF_GRAM) {
          tma_load_2d(sa, tmX, 16 * c, ti * kDfT, &full[s]);
          tma_load_2d(sa + 8192, tmX, 16 * c, tj * kDfT, &full[s]);
        } else {
          tma_load_2d(sa, tmA, ta * kDfT + 16 * c, ti * kDfT, &full[s]);
          tma_load_2d(sa + 8192, tmA, ta * kDfT + 16 * c, tj * kDfT, &full[s]);
        }
      }
    }
  }

  // ---------------- DMMA warps (2 x 2 grid, 32 x 32 each) ----------------
  const int wm = warp >> 1, wn = warp & 1;
  const int lr = lane >> 2, lk = lane & 3;
  int kt = 0;
  for (int it = 0;; ++it) {
    const int slot = it & 1;
    const uint32_t ph = (it >> 1) & 1;
    mbar_wait(&tfull[slot], ph);
    const int4 task = tslot[slot];
#ifdef PKRR_DF_TRACE
    const int ticket = tticket[slot];
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive(&tempty[slot]);
    if (tid == 0) {  // the publisher's copy (its slot is free once task it - 2 is published)
      mbar_wait(&pubempty[slot], ph ^ 1);
      ptask[slot] = task;
#ifdef PKRR_DF_TRACE
      pticket[slot] = ticket;
#endif
    }
    if (task.x == DF_END) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&pubfull[slot]);
      return;
    }
    const int ti = task.y, tj = task.z, ta = task.w & 0xffff, tb = task.w >> 16;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int nk =
        task.x == DF_TRSM ? 4 : (task.x == DF_UPD ? 4 * (tb - ta) : (task.x == DF_GRAM ? p.xk : 0));
    for (int c = 0; c < nk; ++c, ++kt) {
      const int s = kt % kDfStages;
      mbar_wait(&full[s], (kt / kDfStages) & 1);
      if (c > 0) {  // deferred release (see gemm_dmma.cuh)
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[(kt - 1) % kDfStages]);
      }
      const unsigned char* sa = ring + s * kDfStage;
      const unsigned char* sb = sa + 8192;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int k = ks * 4 + lk;
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = lds_f64(sa, swz128(wm * 32 + i * 8 + lr, k));
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = lds_f64(sb, swz128(wn * 32 + j * 8 + lr, k));
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
    }
    if (nk > 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[(kt - 1) % kDfStages]);
    }
    mbar_wait(&cfull[slot], ph);
    unsigned char* cb = cbuf + slot * kDfCbuf;
    const int64_t lda = p.lda;
    if (task.x == DF_UPD) {
      double* Cg = p.A + static_cast<int64_t>(ti * kDfT) * lda + tj * kDfT;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = wm * 32 + i * 8 + lr, c = wn * 32 + j * 8 + 2 * lk;
          double2 v = lds_f64x2(smem_u32(cb + (c >> 4) * 8192) + swz128(r, c & 15));
          v.x -= acc[i][j][0];
          v.y -= acc[i][j][1];
          *reinterpret_cast<double2*>(Cg + static_cast<int64_t>(r) * lda + c) = v;
        }
    } else if (task.x == DF_GRAM) {
      // the gram epilogue of dgemm_tn_kernel<G_GRAM_SYM> (kernel.cpp:52-56): dist2 =
      // (n_i + n_j) - 2 x_i.x_j clamped at 0, exp(dist2 * -1/((2 s) s)); unit diagonal,
      // padding rows / columns identity; A = K + shift I
      double* Kg = p.K + static_cast<int64_t>(ti * kDfT) * lda + tj * kDfT;
      double* Ag = p.A + static_cast<int64_t>(ti * kDfT) * lda + tj * kDfT;
      double nb[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = wn * 32 + j * 8 + 2 * lk;
        nb[j][0] = __ldg(p.xnorm + tj * kDfT + c);
        nb[j][1] = __ldg(p.xnorm + tj * kDfT + c + 1);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = wm * 32 + i * 8 + lr, gi = ti * kDfT + r;
        const double na = __ldg(p.xnorm + gi);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = wn * 32 + j * 8 + 2 * lk;
          double v[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int gj = tj * kDfT + c + e;
            if (gi >= p.m_valid || gj >= p.m_valid) {
              v[e] = gi == gj ? 1.0 : 0.0;
            } else if (gi == gj) {
              v[e] = 1.0;
            } else {
              double dist2 = (na + nb[j][e]) - 2.0 * acc[i][j][e];
              if (dist2 < 0.0) dist2 = 0.0;
              v[e] = exp_nonpos(dist2 * p.neg_inv_denom);
            }
          }
          *reinterpret_cast<double2*>(Kg + static_cast<int64_t>(r) * lda + c) = make_double2(v[0], v[1]);
          const int gj0 = tj * kDfT + c;
          *reinterpret_cast<double2*>(Ag + static_cast<int64_t>(r) * lda + c) =
              make_double2(gi == gj0 ? v[0] + p.shift : v[0], gi == gj0 + 1 ? v[1] + p.shift : v[1]);
        }
      }
    } else if (task.x == DF_TRSM) {
      double* Cg = p.A + static_cast<int64_t>(ti * kDfT) * lda + tj * kDfT;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = wm * 32 + i * 8 + lr, c = wn * 32 + j * 8 + 2 * lk;
          *reinterpret_cast<double2*>(Cg + static_cast<int64_t>(r) * lda + c) =
              make_double2(acc[i][j][0], acc[i][j][1]);
        }
      if (p.z) {
        // this tile's share of the forward substitution, P[ti][tj] = L(ti,tj) z_tj:
        // per-thread partials over its columns, the 4 lanes of a row, then the 4 column
        // warps in a fixed order (deterministic)
        double zc[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          zc[j][0] = __ldcg(p.z + tj * kDfT + wn * 32 + j * 8 + 2 * lk);
          zc[j][1] = __ldcg(p.z + tj * kDfT + wn * 32 + j * 8 + 2 * lk + 1);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double part = 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) part = fma(acc[i][j][1], zc[j][1], fma(acc[i][j][0], zc[j][0], part));
          part += __shfl_xor_sync(0xffffffffu, part, 1);
          part += __shfl_xor_sync(0xffffffffu, part, 2);
          if (lk == 0) red[wn * 64 + wm * 32 + i * 8 + lr] = part;
        }
        consumer_sync(128);
        if (tid < 64) p.P[(static_cast<int64_t>(ti) * nt + tj) * kDfT + tid] = red[tid] + red[64 + tid];
        consumer_sync(128);  // red is read: the next TRSM may overwrite it
      }
    } else {
      // DF_INV: the 128 x 128 diagonal-block inverse [X0 0; Y X1] of block pair ti,
      // Y = -X1 (L21 X0), for the backward solve (trsv_bwd_kernel reads Linv)
      const int b2 = 2 * ti;
      const double* L21 = p.A + static_cast<int64_t>((b2 + 1) * kDfT) * lda + b2 * kDfT;
      const double* X0 = p.inv64 + static_cast<int64_t>(b2) * 4096;
      const double* X1 = X0 + 4096;
      double* T1 = reinterpret_cast<double*>(cb);  // [64][64]
#pragma unroll 4
      for (int k = 0; k < 64; k += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = __ldcg(L21 + static_cast<int64_t>(wm * 32 + i * 8 + lr) * lda + k + lk);
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = __ldcg(X0 + (k + lk) * 64 + wn * 32 + j * 8 + lr);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = wm * 32 + i * 8 + lr, c = wn * 32 + j * 8 + 2 * lk;
          T1[r * 64 + c] = acc[i][j][0];
          T1[r * 64 + c + 1] = acc[i][j][1];
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
      consumer_sync(128);
#pragma unroll 4
      for (int k = 0; k < 64; k += 4) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = __ldcg(X1 + (wm * 32 + i * 8 + lr) * 64 + k + lk);
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = T1[(k + lk) * 64 + wn * 32 + j * 8 + lr];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
      double* Lo = p.Linv + static_cast<int64_t>(ti) * 128 * 128;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = wm * 32 + i * 8 + lr, c = wn * 32 + j * 8 + 2 * lk;
          *reinterpret_cast<double2*>(Lo + (64 + r) * 128 + c) = make_double2(-acc[i][j][0], -acc[i][j][1]);
        }
      for (int e = tid; e < 64 * 32; e += 128) {
        const int r = e >> 5, c2 = 2 * (e & 31);
        *reinterpret_cast<double2*>(Lo + r * 128 + c2) = __ldcg(reinterpret_cast<const double2*>(X0 + r * 64 + c2));
        *reinterpret_cast<double2*>(Lo + r * 128 + 64 + c2) = make_double2(0.0, 0.0);
        *reinterpret_cast<double2*>(Lo + (64 + r) * 128 + 64 + c2) =
            __ldcg(reinterpret_cast<const double2*>(X1 + r * 64 + c2));
      }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&cempty[slot]);
      mbar_arrive(&pubfull[slot]);  // this warp's stores are issued: the publisher releases the task
    }
  }
}

// ---------------------------------------------------------------------------
// chain CTA
// ---------------------------------------------------------------------------
// Compact reciprocal / reciprocal square root (MUFU approximation + two Newton steps;
// x is a positive normal pivot).  Inline-expanded library versions carry special-case
// paths that multiply the chain's code size, and the chain must stay inside the SM's
// 32 KB L1.5 instruction cache (the unrolled 128-leaf ran instruction-fetch bound).
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  // MUFU seed + one Halley step (cubic): y (1 + e/2 + 3e^2/8), e = 1 - x y^2
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

// Per 32-column panel of a 64-column chain step, one warp factors the 32 x 32
// diagonal block in ROW layout (lane i owns row i, a[c] = S[i][c]): the reference's
// column loop (solver.cpp:18-33) -- pivot test, scale, rank-1 update -- per column j.
// The pivot chain is SHFL -> rsqrt -> multiply -> FMA -> SHFL: lane j+1's next pivot
// a[j+1] - l^2 and its column value travel by SHFL; the column values and rsqrt(pivot)
// go to slot j of `ds` (33 slots of 40 doubles: [0, 32) the column, [33] the rsqrt)
// with mbarrier cbar[j], for the rest of the update and for the warps factoring rows
// below the diagonal block (warp_tall32s), which follow one column behind at most, or
// later (every slot of the panel stays valid for the whole step).  Straight-line code
// (the scheduler interleaves the update with the pivot chain).  Returns the first
// failing pivot column, or -1.
template <int LS>
__device__ __noinline__ int warp_diag32(uint32_t S, uint32_t Xs, uint32_t ds, int lane) {
  // S: the 32 x 32 diagonal block (factored in place, rows = lanes); Xs: 32 x 32 rows of
  // the identity, turned into X = L^{-T} by the same column loop (the panel TRSM of the
  // reference's loop applied to unit rows): inv(L) = X^T without a separate inversion.
  // Rolled over 4 groups of 8 columns; the row registers rotate by 8 per group so the
  // group's columns are always a[0..7] (a few KB of code: the loop stays resident in
  // the instruction cache while the other warps' DMMA loops run beside it).
  double a[32], x[32];
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    const double2 v = lds_f64x2(S + (lane * LS + c) * 8);
    a[c] = v.x;
    a[c + 1] = v.y;
    x[c] = c == lane ? 1.0 : 0.0;
    x[c + 1] = c + 1 == lane ? 1.0 : 0.0;
  }
  int bad = -1;
  double piv = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll 1
  for (int g = 0; g < 4; ++g) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = 8 * g + c;  // global column
      const uint32_t slot = ds + j * 256;
      if (!(piv > 0.0) && bad < 0) bad = j;
      const double r = rsqrt_nr(bad >= 0 ? 1.0 : piv);
      const double l = a[c] * r, lx = x[c] * r;
      // lane j+1's next pivot and column value (j + 1 == 32 reads a dead value)
      piv = __shfl_sync(0xffffffffu, fma(-l, l, a[c + 1]), (j + 1) & 31);
      const double ln = __shfl_sync(0xffffffffu, l, (j + 1) & 31);
      sts_f64(slot + lane * 8, l);
      __syncwarp();
      sts_f64(S + (lane * LS + j) * 8, lane >= j ? l : 0.0);  // final L and X column j
      sts_f64(Xs + (lane * LS + j) * 8, lx);
      a[c + 1] = fma(-l, ln, a[c + 1]);
      x[c + 1] = fma(-lx, ln, x[c + 1]);
      // columns j + 2 .. (registers c + 2 .. 31; those past column 31 hold dead values)
#pragma unroll
      for (int k = c + 2; k < 32; ++k) {
        const double v = lds_f64_at(slot + ((j + k - c) & 31) * 8);
        a[k] = fma(-l, v, a[k]);
        x[k] = fma(-lx, v, x[k]);
      }
    }
#pragma unroll
    for (int i = 0; i < 24; ++i) {
      a[i] = a[i + 8];
      x[i] = x[i + 8];
    }
  }
  return bad;
}

// Fully unrolled variant of warp_diag32 (the default; PKRR_DF_ROLLED selects the rolled
// one): straight-line code, fewer instructions per column (6.9K vs 9.6K cycles per
// 32-column panel alone), ~28 KB streamed through the instruction cache per call --
// measured 1.60 vs 1.63 ms for a 4096-row system.
template <int LS>
__device__ __noinline__ int warp_diag32u(uint32_t S, uint32_t Xs, uint32_t ds, int lane) {
  double a[32], x[32];
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    const double2 v = lds_f64x2(S + (lane * LS + c) * 8);
    a[c] = v.x;
    a[c + 1] = v.y;
    x[c] = c == lane ? 1.0 : 0.0;
    x[c + 1] = c + 1 == lane ? 1.0 : 0.0;
  }
  int bad = -1;
  double piv = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const uint32_t slot = ds + j * 256;
    if (!(piv > 0.0) && bad < 0) bad = j;
    const double r = rsqrt_nr(bad >= 0 ? 1.0 : piv);
    const double l = a[j] * r, lx = x[j] * r;
    double ln = 0.0;
    if (j + 1 < 32) {
      piv = __shfl_sync(0xffffffffu, fma(-l, l, a[j + 1]), j + 1);
      ln = __shfl_sync(0xffffffffu, l, j + 1);
    }
    sts_f64(slot + lane * 8, l);
    __syncwarp();
    a[j] = lane >= j ? l : 0.0;
    x[j] = lx;
    if (j + 1 < 32) {
      a[j + 1] = fma(-l, ln, a[j + 1]);
      x[j + 1] = fma(-lx, ln, x[j + 1]);
    }
    int k = j + 2;
    if (k < 32 && (k & 1)) {
      const double v = lds_f64_at(slot + k * 8);
      a[k] = fma(-l, v, a[k]);
      x[k] = fma(-lx, v, x[k]);
      ++k;
    }
#pragma unroll
    for (; k < 32; k += 2) {
      const double2 v = lds_f64x2(slot + k * 8);
      a[k] = fma(-l, v.x, a[k]);
      a[k + 1] = fma(-l, v.y, a[k + 1]);
      x[k] = fma(-lx, v.x, x[k]);
      x[k + 1] = fma(-lx, v.y, x[k + 1]);
    }
  }
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    sts_f64x2(S + (lane * LS + c) * 8, make_double2(a[c], a[c + 1]));
    sts_f64x2(Xs + (lane * LS + c) * 8, make_double2(x[c], x[c + 1]));
  }
  return bad;
}
#ifdef PKRR_DF_ROLLED
#define DF_DIAG warp_diag32
#else
#define DF_DIAG warp_diag32u
#endif

__device__ __forceinline__ void df_record_npd(const DfParams& p, int col, int* sflag) {
  *sflag = 1;
  p.status[1] = col;
  __threadfence();
  atomicExch(&p.status[0], 1);
}

// The chain's small products are dependent-DMMA-latency bound (one accumulator chain of
// K / 4 steps per 8 x 8 tile), so K is split SPLIT ways into independent chains that are
// summed at the end in a fixed order (kDfSplit k-ranges of K / kDfSplit).
#ifndef PKRR_DF_SPLIT
#define PKRR_DF_SPLIT 0
#endif
// rows [16 rb, 16 rb + 16) x cols [16 cb, +16) of dst -= A(rows) B(cols)^T over K (16 x 16
// blocks of 2 x 2 DMMA tiles); lower_diag skips the strictly upper 8 x 8 tile of a
// diagonal block
__device__ __forceinline__ void df_block_update(double* dst, const double* Arow, const double* Brow, int K,
                                                bool lower_diag, int lr, int lk) {
#if PKRR_DF_SPLIT
  double part[4][2][2][2] = {};
  const int KS = K >> 2;
#pragma unroll 2
  for (int k = 0; k < KS; k += 4) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int kk = s * KS + k + lk;
      const double a0 = Arow[lr * kDS + kk], a1 = Arow[(8 + lr) * kDS + kk];
      const double b0 = Brow[lr * kDS + kk], b1 = Brow[(8 + lr) * kDS + kk];
      dmma(part[s][0][0], a0, b0);
      dmma(part[s][0][1], a0, b1);
      dmma(part[s][1][0], a1, b0);
      dmma(part[s][1][1], a1, b1);
    }
  }
  double acc[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        acc[i][j][e] = (part[0][i][j][e] + part[1][i][j][e]) + (part[2][i][j][e] + part[3][i][j][e]);
#else
  double acc[2][2][2] = {};
  mma_2x2_rt(acc, Arow, Brow, kDS, K, lr, lk);
#endif
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (lower_diag && j > i) continue;
      double* d2 = dst + (8 * i + lr) * kDS + 8 * j + 2 * lk;
      const double2 v = *reinterpret_cast<double2*>(d2);
      *reinterpret_cast<double2*>(d2) = make_double2(v.x - acc[i][j][0], v.y - acc[i][j][1]);
    }
}

// 8-row x 32-column DMMA items of the chain's small products (row-major operands with
// the chain stride): C (=, -=) A(8 rows, K) . B(K, 32) ["rn"] or A . Bt(32 rows, K)^T ["rt"]
__device__ __forceinline__ void df_store8(double* dst, double (&acc)[4][2], int mode, int lr, int lk) {
  // mode 0: dst = acc, 1: dst -= acc, 2: dst = -acc
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double2* d2 = reinterpret_cast<double2*>(dst + lr * kDS + 8 * c + 2 * lk);
    if (mode == 1) {
      const double2 v = *d2;
      *d2 = make_double2(v.x - acc[c][0], v.y - acc[c][1]);
    } else {
      *d2 = mode == 0 ? make_double2(acc[c][0], acc[c][1]) : make_double2(-acc[c][0], -acc[c][1]);
    }
  }
}
__device__ __forceinline__ void df_rn8(double* dst, const double* A, const double* B, int mode, int lr, int lk) {
  double acc[4][2] = {};
#if PKRR_DF_SPLIT
  double p1[4][2] = {};  // K = 32 as two chains of 4 steps
#pragma unroll 2
  for (int k = 0; k < 16; k += 4) {
    const double a0 = A[lr * kDS + k + lk], a1 = A[lr * kDS + 16 + k + lk];
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma(acc[c], a0, B[(k + lk) * kDS + 8 * c + lr]);
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma(p1[c], a1, B[(16 + k + lk) * kDS + 8 * c + lr]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    acc[c][0] += p1[c][0];
    acc[c][1] += p1[c][1];
  }
#else
  mma_row4_rn(acc, A, kDS, B, kDS, 0, 32, lr, lk);
#endif
  __syncwarp();  // in place: every read of these rows precedes the write
  df_store8(dst, acc, mode, lr, lk);
}
__device__ __forceinline__ void df_rt8(double* dst, const double* A, const double* Bt, int K, int mode, int lr,
                                      int lk) {
  double acc[4][2] = {};
#if PKRR_DF_SPLIT
  double p1[4][2] = {};  // two chains of K / 8 steps
  const int KS = K >> 1;
#pragma unroll 2
  for (int k = 0; k < KS; k += 4) {
    const double a0 = A[lr * kDS + k + lk], a1 = A[lr * kDS + KS + k + lk];
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma(acc[c], a0, Bt[(8 * c + lr) * kDS + k + lk]);
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma(p1[c], a1, Bt[(8 * c + lr) * kDS + KS + k + lk]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    acc[c][0] += p1[c][0];
    acc[c][1] += p1[c][1];
  }
#else
  mma_row4_rt(acc, A, kDS, Bt, kDS, 0, K, lr, lk);
#endif
  __syncwarp();
  df_store8(dst, acc, mode, lr, lk);
}

// dst8 (8 x 32) -= A8 (8 rows, K = 64) . Bt(32 rows)^T  and  the lower 16 x 16 block
// dst16 -= S(16 rows) . S^T, in one k loop
__device__ __forceinline__ void df_rt8_block11(double* dst8, double* dst16, const double* A8, const double* Bt,
                                               const double* S, int lr, int lk) {
  double acc[4][2] = {}, b00[2] = {}, b10[2] = {}, b11[2] = {};
#pragma unroll 4
  for (int k = 0; k < 64; k += 4) {
    const double a = A8[lr * kDS + k + lk];
    const double s0 = S[lr * kDS + k + lk], s1 = S[(8 + lr) * kDS + k + lk];
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma(acc[c], a, Bt[(8 * c + lr) * kDS + k + lk]);
    dmma(b00, s0, s0);
    dmma(b10, s1, s0);
    dmma(b11, s1, s1);
  }
  __syncwarp();
  df_store8(dst8, acc, 1, lr, lk);
  double2* d = reinterpret_cast<double2*>(dst16 + lr * kDS + 2 * lk);
  double2 v = *d;
  *d = make_double2(v.x - b00[0], v.y - b00[1]);
  d = reinterpret_cast<double2*>(dst16 + (8 + lr) * kDS + 2 * lk);
  v = *d;
  *d = make_double2(v.x - b10[0], v.y - b10[1]);
  d = reinterpret_cast<double2*>(dst16 + (8 + lr) * kDS + 8 + 2 * lk);
  v = *d;
  *d = make_double2(v.x - b11[0], v.y - b11[1]);
}

// The chain's tile loads, issued by one thread without holding up the step's barriers:
// polled (non-blocking) at the phase boundaries, waited for only where the data is used.
// The chain's tile loads come from warp 4 alone, which never joins the step's barriers:
// issuing the 64 row copies of a tile costs microseconds (~30 ns per cp.async.bulk), so
// a loader inside a barrier would stall the whole step.  Per step k it waits until the
// compute warps have started the step (stepbar: the buffers are free), then issues T(k)
// = tile (k+1, k) and D(k+1) = tile (k+1, k+1) as soon as the workers have applied
// panels [0, k) to each (tbar / lbar complete_tx), whichever is ready first.
__device__ __forceinline__ bool df_tile_load(const DfParams& p, const int* flag, int target, double* dst,
                                             const double* src, uint64_t* bar, int lane) {
  int ready = 0;
  if (lane == 0) ready = *reinterpret_cast<const volatile int*>(flag) >= target;
  ready = __shfl_sync(0xffffffffu, ready, 0);
  if (!ready) return false;
  if (lane == 0) mbar_arrive_expect_tx(bar, 64 * 512);
  __syncwarp();
  (void)ld_acquire_gpu(flag);
  fence_proxy_async_global();
  const int64_t lda = p.lda;
  bulk_load(dst + lane * kDS, src + static_cast<int64_t>(lane) * lda, 512, bar);
  bulk_load(dst + (lane + 32) * kDS, src + static_cast<int64_t>(lane + 32) * lda, 512, bar);
  return true;
}
__device__ __noinline__ void df_loader(const DfParams& p, double* Dbuf, double* Tbuf, uint64_t* lbar, uint64_t* tbar,
                                       uint64_t* stepbar, int lane) {
  const int nt = p.nt;
  const int* applied = p.flags + F_HEAD;
  const int64_t lda = p.lda;
  for (int k = 0; k + 1 < nt; ++k) {
    // a sleeping wait: this warp shares its scheduler partition with the diagonal warp,
    // and a try_wait spin takes issue slots from it for the whole first panel
    while (!mbar_test(stepbar, k & 1)) {
      if (*reinterpret_cast<const volatile int*>(p.status)) return;  // the chain abandoned (NPD)
      __nanosleep(128);
    }
    bool dd = false, td = false;
    const long long t0 = clock64();
    while (!(dd && td)) {
      if (!td)
        td = df_tile_load(p, applied + (k + 1) * nt + k, k, Tbuf + (k & 1) * 64 * kDS,
                          p.A + static_cast<int64_t>((k + 1) * kDfT) * lda + k * kDfT, tbar, lane);
      if (!dd)
        dd = df_tile_load(p, applied + (k + 1) * nt + (k + 1), k, Dbuf + ((k + 1) & 1) * 64 * kDS,
                          p.A + static_cast<int64_t>((k + 1) * kDfT) * lda + (k + 1) * kDfT, lbar, lane);
      if (!(dd && td)) {
        if (__shfl_sync(0xffffffffu, *reinterpret_cast<const volatile int*>(p.status), 0)) return;
        if (clock64() - t0 > (1ll << 33)) __trap();
        __nanosleep(64);
      }
    }
  }
}

// One chain step k (64 columns).  Warp 0 runs the column-sequential work; everything
// else is placed so that it overlaps warp 0 wherever the dependencies allow:
//   [A] warp 0: D00 -> L00, X00 = L00^{-T}.  Helpers (warps 1-3, 5-7), finishing step k-1
//       beside it: T(k-1) rows 32..63 T1 X11(k-1) -> publish L(k,k-1) (lrow[k]),
//       P[k][k-1] = L(k,k-1) z_{k-1}, w_k; D(k) rows 32..63 -= L(k,k-1)[32:] L(k,k-1)^T;
//       store L_{k-1}; then the loader may refill D(k-1) / T(k-2)'s buffers (stepbar).
//   [B] L10 = D10 X00
//   [C] warp 0: D11 -> L11, X11 (after D11 -= L10 L10^T by warps 1-3); Xtmp = X00 L10^T;
//       T(k) rows (if they arrived): T0 X00, T1 -= T0 L10^T
//   [D] X01 = -Xtmp X11; z_k = X^T w_k; publish inv(L_kk) = X^T, z_k (chain = k + 1)
//   [E] T(k) rows: the rest of T0 X00 / T1 -= T0 L10^T, and T1 X11 for rows 0..31;
//       D(k+1)00 -= T(k)[:32] T(k)[:32]^T, the block the next step's warp 0 starts on.
__device__ __forceinline__ void df_chain(const DfParams& p, unsigned char* smem) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int lr = lane >> 2, lk = lane & 3;
  const int nt = p.nt;
  const int64_t lda = p.lda;
  double* Dbuf = reinterpret_cast<double*>(smem);  // 2 x [64][kDS]: diagonal tiles k, k+1
  double* Tbuf = Dbuf + 2 * 64 * kDS;              // 2 x [64][kDS]: tiles (k+1, k), (k, k-1)
  double* X = Tbuf + 2 * 64 * kDS;                 // X = L_kk^{-T} (upper triangular; X10 stays 0)
  double* ds = X + 64 * kDS;                       // diagonal warp's 32 column slots of 32
  double* wv = ds + 32 * 32;
  double* zv = wv + 64;
  double* pv = zv + 64;    // P[k][k-1] (computed at the start of step k)
  double* red = pv + 64;   // [2][64] partial GEMV sums
  uint64_t* lbar = reinterpret_cast<uint64_t*>(red + 128);
  uint64_t* tbar = lbar + 1;
  uint64_t* dbar = tbar + 1;     // D11 updated by the first panel (warps 1, 2, 3)
  uint64_t* stepbar = dbar + 1;  // step k's helpers are done with D(k-1) / T(k-2): loader may refill
  int* sflag = reinterpret_cast<int*>(stepbar + 1);
  int* tdone = sflag + 1;  // [8] T row tile q has had T0 X00 and T1 -= T0 L10^T
  int* applied = p.flags + F_HEAD;
  int* lrow = applied + nt * nt;
  if (tid == 0) {
    mbar_init(lbar, 1);
    mbar_init(tbar, 1);
    mbar_init(dbar, 3);
    mbar_init(stepbar, 1);
    fence_mbar_init();
    *sflag = 0;
  }
  for (int e = tid; e < 64 * kDS; e += kDfThreads) X[e] = 0.0;
  __syncthreads();
  if (warp == 4) {
    df_loader(p, Dbuf, Tbuf, lbar, tbar, stepbar, lane);
    return;
  }
  // compute warps 0-3, 5-7 (cw 0..6, ctid 0..223) on named barrier 2; the helpers
  // (warps 1-3, 5-7: hw 0..5, htid 0..191) on named barrier 3
  const int cw = warp < 4 ? warp : warp - 1, ctid = cw * 32 + lane;
  const int hw = cw - 1, htid = ctid - 32;
  auto csync = [] { asm volatile("bar.sync 2, 224;\n" ::: "memory"); };
  auto hsync = [] { asm volatile("bar.sync 3, 192;\n" ::: "memory"); };
  if (ctid == 0) {
    df_wait_ge(applied, 0, p.status);  // tile (0, 0) formed (fused gram)
    fence_proxy_async_global();
    mbar_arrive_expect_tx(lbar, 64 * 512);
    for (int r = 0; r < 64; ++r) bulk_load(Dbuf + r * kDS, p.A + static_cast<int64_t>(r) * lda, 512, lbar);
  }
  mbar_wait(lbar, 0);
  const uint32_t uds = smem_u32(ds);
  double* X01 = X + 32;
  double* X11 = X + 32 * kDS + 32;

  for (int k = 0; k < nt; ++k) {
    double* D = Dbuf + (k & 1) * 64 * kDS;
    double* D10 = D + 32 * kDS;
    double* D11 = D10 + 32;
    double* Dp = Dbuf + ((k + 1) & 1) * 64 * kDS;  // D(k-1) = L_{k-1}
    double* T = Tbuf + (k & 1) * 64 * kDS;         // T(k) = tile (k+1, k)
    double* Tp = Tbuf + ((k + 1) & 1) * 64 * kDS;  // T(k-1) = L(k, k-1)
    const bool has_t = k + 1 < nt;
    const uint32_t par = k & 1;
    DF_CHAIN_MARK(k, 0)
#ifdef PKRR_DF_TRACE
    if (threadIdx.x == 0) g_df_chain[k][11] = df_now();
#endif
    // ---------------- [A] ----------------
    int bad = -1;
#ifdef PKRR_DF_TRACE
    if (lane == 0) g_df_warp[k][warp][0] = df_clk();
#endif
    if (warp == 0) {
      __syncwarp();  // converged entry (the callee's SHFLs)
      bad = DF_DIAG<kDS>(smem_u32(D), smem_u32(X), uds, lane);
#ifdef PKRR_DF_TRACE
      if (lane == 0) g_df_chain[k][2] = df_clk();
#endif
    } else {
      if (k > 0) {
        // publish L(k, k-1) (finished in step k-1's [E]) first: the worker update of tile
        // (k+1, k) that the chain reloads as T(k) waits for it; P[k][k-1] = L(k,k-1) z_{k-1}
        double* Tg = p.A + static_cast<int64_t>(k * kDfT) * lda + (k - 1) * kDfT;
        for (int e = htid; e < 64 * 32; e += 192) {
          const int r = e >> 5, c2 = 2 * (e & 31);
          *reinterpret_cast<double2*>(Tg + static_cast<int64_t>(r) * lda + c2) =
              *reinterpret_cast<const double2*>(Tp + r * kDS + c2);
        }
        if (p.z && htid < 128) {
          const int r = htid & 63, pt = htid >> 6;
          double sacc = 0.0;
          for (int c = 32 * pt; c < 32 * pt + 32; ++c) sacc = fma(Tp[r * kDS + c], zv[c], sacc);
          red[pt * 64 + r] = sacc;
        }
        hsync();
        if (htid == 0) {
          st_release_gpu(lrow + k, k);
#ifdef PKRR_DF_TRACE
          g_df_warp[k][4][0] = df_now();
#endif
        }
        if (p.z && htid < 64) pv[htid] = red[htid] + red[64 + htid];
        // D(k) rows 32..63 -= L(k,k-1)[32:64] L(k,k-1)^T (K = 64): D10 as 4 row tiles,
        // D11 (lower) as 3 blocks of 16; L_{k-1} to global
        if (hw == 0) {
          // this warp's two items (D10 row tile 0, D11 block (1,1)) as one loop: 7
          // independent DMMA chains instead of two latency-bound passes
          df_rt8_block11(D10, D11 + 16 * kDS + 16, Tp + 32 * kDS, Tp, Tp + 48 * kDS, lr, lk);
        } else for (int t = hw; t < 6; t += 6) {
          if (t < 4) {
            df_rt8(D10 + 8 * t * kDS, Tp + (32 + 8 * t) * kDS, Tp, 64, 1, lr, lk);
          } else {
            const int rb = t == 4 ? 0 : 1, cb = t == 6 ? 1 : 0;
            df_block_update(D11 + 16 * rb * kDS + 16 * cb, Tp + (32 + 16 * rb) * kDS, Tp + (32 + 16 * cb) * kDS,
                            64, rb == cb, lr, lk);
          }
        }
        double* Ag = p.A + static_cast<int64_t>((k - 1) * kDfT) * lda + (k - 1) * kDfT;
        for (int e = htid; e < 64 * 32; e += 192) {
          const int r = e >> 5, c2 = 2 * (e & 31);
          if (c2 <= r)
            *reinterpret_cast<double2*>(Ag + static_cast<int64_t>(r) * lda + c2) =
                *reinterpret_cast<const double2*>(Dp + r * kDS + c2);
        }
      }
#ifdef PKRR_DF_TRACE
      if (lane == 0) g_df_warp[k][warp][1] = df_clk();
#endif
      hsync();  // pv, D(k-1) and T(k-2) done with
      if (htid == 0) {
        fence_proxy_async();
        mbar_arrive(stepbar);  // the loader may refill D(k-1) / T(k-2)'s buffers
      }
      if (htid < 8) tdone[htid] = 0;
    }
#ifdef PKRR_DF_TRACE
    if (lane == 0) g_df_warp[k][warp][5] = df_clk();
#endif
    csync();
    DF_CHAIN_MARK(k, 1)
    // ---------------- [B] L10 = D10 X00 ----------------
    const int dw = warp == 5 ? 3 : warp - 1;  // 0..3 for warps 1, 2, 3, 5
    if (warp == 1 || warp == 2 || warp == 3 || warp == 5) df_rn8(D10 + 8 * dw * kDS, D10 + 8 * dw * kDS, X, 0, lr, lk);
    if (warp == 0 && bad >= 0 && lane == 0) df_record_npd(p, k * kDfT + bad, sflag);
#ifdef PKRR_DF_TRACE
    if (lane == 0) g_df_warp[k][warp][2] = df_clk();
#endif
    csync();
    DF_CHAIN_MARK(k, 3)
    // ---------------- [C] ----------------
    if (warp == 0) {
      mbar_wait(dbar, par);
      __syncwarp();
      const int bad1 = DF_DIAG<kDS>(smem_u32(D11), smem_u32(X11), uds, lane);
      if (bad1 >= 0 && lane == 0 && !*sflag) df_record_npd(p, k * kDfT + 32 + bad1, sflag);
    } else if (warp >= 1 && warp <= 3) {
      const int rb = warp == 1 ? 1 : (warp == 2 ? 0 : 1), cb = warp == 3 ? 1 : 0;
      df_block_update(D11 + 16 * rb * kDS + 16 * cb, D10 + 16 * rb * kDS, D10 + 16 * cb * kDS, 32, rb == cb, lr, lk);
      __syncwarp();
      if (lane == 0) mbar_arrive(dbar);
      for (int q = warp - 1; q < 4; q += 3) df_rt8(X01 + 8 * q * kDS, X + 8 * q * kDS, D10, 32, 0, lr, lk);
    } else if (warp >= 5) {
      if (p.z && warp >= 6) {
        // w_k = y_k - sum_p P[k][p] in panel order (P[k][k-1] = pv from [A]); the P loads are
        // L2 round trips, so they run here, beside the second diagonal panel, not on the
        // way to a barrier of the chain
        const int r = lane + 32 * (warp - 6);
        double sw = p.y[k * kDfT + r];
        const double* pk_ = p.P + static_cast<int64_t>(k) * nt * kDfT + r;
        int q = 0;
        for (; q + 8 <= k - 1; q += 8) {
          double a[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) a[u] = __ldcg(pk_ + (q + u) * kDfT);
#pragma unroll
          for (int u = 0; u < 8; ++u) sw -= a[u];
        }
        for (; q < k - 1; ++q) sw -= __ldcg(pk_ + q * kDfT);
        if (k > 0) sw -= pv[r];
        wv[r] = sw;
      }
      if (has_t && __shfl_sync(0xffffffffu, mbar_test(tbar, par), 0)) {
        for (int q = warp - 5; q < 8; q += 3) {
          df_rn8(T + 8 * q * kDS, T + 8 * q * kDS, X, 0, lr, lk);
          __syncwarp();
          df_rt8(T + 8 * q * kDS + 32, T + 8 * q * kDS, D10, 32, 1, lr, lk);
          if (lane == 0) tdone[q] = 1;
        }
      }
    }
#ifdef PKRR_DF_TRACE
    if (lane == 0) g_df_warp[k][warp][3] = df_clk();
#endif
    csync();
    DF_CHAIN_MARK(k, 4)
    // ---------------- [D] X01, z_k, publish inv(L_kk), z_k ----------------
    if (warp < 4) df_rn8(X01 + 8 * warp * kDS, X01 + 8 * warp * kDS, X11, 2, lr, lk);
#ifdef PKRR_DF_TRACE
    if (lane == 0) g_df_warp[k][warp][4] = df_clk();
#endif
    csync();
    if (*sflag) return;
    DF_CHAIN_MARK(k, 5)
    // ---------------- [E] ----------------
    // critical (warps 0-3): rows 0..31 of T(k) (all three products) and then D(k+1)00, the
    // block the next step's diagonal warp starts on.  Background (warps 5-7), beside it:
    // z_k = X^T w_k, publish inv(L_kk) = X^T and z_k (chain = k + 1: the fence's L2 round
    // trip is off the critical warps), then rows 32..55 of T(k); rows 56..63 go to warp 3
    // beside the D(k+1)00 update.  T(k) = L(k+1, k) is complete at the end of the step, so
    // the next step's [A] publishes it at once.
    auto trow = [&](int q) {
      if (!tdone[q]) {
        df_rn8(T + 8 * q * kDS, T + 8 * q * kDS, X, 0, lr, lk);
        __syncwarp();
        df_rt8(T + 8 * q * kDS + 32, T + 8 * q * kDS, D10, 32, 1, lr, lk);
      }
      __syncwarp();
      df_rn8(T + 8 * q * kDS + 32, T + 8 * q * kDS + 32, X11, 0, lr, lk);
    };
    if (warp >= 5) {
      const int bt = (warp - 5) * 32 + lane;
      if (p.z && bt < 64) {
        double s0 = 0.0, s1 = 0.0;  // the two half sums, then their sum (fixed order)
#pragma unroll 8
        for (int c = 0; c < 32; ++c) {
          s0 = fma(X[c * kDS + bt], wv[c], s0);
          s1 = fma(X[(c + 32) * kDS + bt], wv[c + 32], s1);
        }
        const double z = s0 + s1;
        zv[bt] = z;
        p.z[k * kDfT + bt] = z;
      }
      double* Ig = p.inv64 + static_cast<int64_t>(k) * 4096;
      for (int e = bt; e < 64 * 32; e += 96) {
        const int ri = e & 63, ci = 2 * (e >> 6);  // X read down its columns: conflict-free
        *reinterpret_cast<double2*>(Ig + ri * 64 + ci) = make_double2(X[ci * kDS + ri], X[(ci + 1) * kDS + ri]);
      }
      asm volatile("bar.sync 5, 96;\n" ::: "memory");
      if (bt == 0) {
        st_release_gpu(p.flags + F_CHAIN, k + 1);
#ifdef PKRR_DF_TRACE
        g_df_chain[k][9] = df_now();
#endif
      }
#ifdef PKRR_DF_TRACE
      if (lane == 0) g_df_warp[k][warp][6] = df_clk();
#endif
      if (has_t) {
        mbar_wait(tbar, par);
        trow(warp - 1);
      }
#ifdef PKRR_DF_TRACE
      if (lane == 0) g_df_warp[k][warp][7] = df_clk();
#endif
    } else if (has_t) {
      mbar_wait(tbar, par);
      DF_CHAIN_MARK(k, 7)
      trow(warp);
#ifdef PKRR_DF_TRACE
      if (lane == 0) g_df_warp[k][warp][7] = df_clk();
#endif
      mbar_wait(lbar, (k + 1) & 1);  // D(k+1) prefetched
      asm volatile("bar.sync 4, 128;\n" ::: "memory");
      DF_CHAIN_MARK(k, 8)
      if (warp < 3) {
        double* Dn = Dbuf + ((k + 1) & 1) * 64 * kDS;
        const int rb = warp == 0 ? 0 : 1, cb = warp == 2 ? 1 : 0;
        df_block_update(Dn + 16 * rb * kDS + 16 * cb, T + 16 * rb * kDS, T + 16 * cb * kDS, 64, rb == cb, lr, lk);
      } else {
        trow(7);
      }
    }
    csync();
    if (!has_t) break;
    DF_CHAIN_MARK(k, 10)
  }
  // the last diagonal block
  {
    const int k = nt - 1;
    double* D = Dbuf + (k & 1) * 64 * kDS;
    double* Ag = p.A + static_cast<int64_t>(k * kDfT) * lda + k * kDfT;
    for (int e = ctid; e < 64 * 32; e += 224) {
      const int r = e >> 5, c2 = 2 * (e & 31);
      if (c2 <= r)
        *reinterpret_cast<double2*>(Ag + static_cast<int64_t>(r) * lda + c2) =
            *reinterpret_cast<const double2*>(D + r * kDS + c2);
    }
  }
}

__global__ void __launch_bounds__(kDfThreads, 1)
    potrf_df_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmI,
                    const __grid_constant__ CUtensorMap tmX, DfParams p) {
  if (*reinterpret_cast<const volatile int*>(p.status)) return;
  extern __shared__ unsigned char df_smem_raw[];
  // 1024-byte alignment (128B-swizzled TMA ring) by pointer arithmetic on the shared
  // array itself, so the compiler keeps the shared address space (LDS / STS, not
  // generic LD / ST) through every derived pointer
  unsigned char* smem = df_smem_raw + ((1024u - (smem_u32(df_smem_raw) & 1023u)) & 1023u);
  __shared__ int role;
  if (threadIdx.x == 0) role = atomicAdd(p.flags + F_ROLE, 1);
  __syncthreads();
  if (role == 0)
    df_chain(p, smem);
  else
    df_worker(&tmA, &tmI, &tmX, p, smem);
}

}  // namespace pk
