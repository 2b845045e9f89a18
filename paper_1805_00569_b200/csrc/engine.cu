// engine.cu -- host side of the B200 pkrr engine: the C ABI of include/pkrr_gpu.h.
//
// Mirrors the reference's 4-stage API (strategies.hpp:40-120): partition ->
// per-part train -> best-cell select -> predict, with the reference's argument
// meaning and error semantics.  All arithmetic runs in the sm_100a kernels of
// kernels.cu / gemm_dmma.cuh; the host only sequences launches, draws the
// k-means init permutation with the reference's RNG (rng.cpp), and runs the
// O(k) control decisions of the clustering loops (convergence, empty-cluster
// reseed, k-balance capacity bookkeeping) exactly as clustering.cpp does.
#include <algorithm>
#include <cctype>
#include <memory>
#include <thread>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <random>
#include <string>
#include <vector>
#include <array>

#include "../../include/pkrr_gpu.h"
#include "kernels.cuh"

using pk::kNB;

namespace {

thread_local std::string g_err;

struct Fail {
  int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
  g_err = msg;
  throw Fail{code};
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(PKRRGPU_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ---- reference RNG (rng.hpp:14-42, rng.cpp:8-63): host side, init only ----
class HostRng {
 public:
  explicit HostRng(uint64_t seed) : eng_(seed) {}
  uint64_t below(uint64_t n) {
    if (n <= 1) return 0;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
      x = eng_();
    } while (x >= limit);
    return x % n;
  }
  std::vector<int64_t> permutation(int64_t n) {
    std::vector<int64_t> perm(n);
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    for (int64_t i = n; i > 1; --i) {
      const int64_t j = static_cast<int64_t>(below(static_cast<uint64_t>(i)));
      std::swap(perm[i - 1], perm[j]);
    }
    return perm;
  }

 private:
  std::mt19937_64 eng_;
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int predictor_of(int s) {
  switch (s) {
    case PKRRGPU_EXACT: return 0;
    case PKRRGPU_DCKRR: case PKRRGPU_KKRR: case PKRRGPU_BKRR: return 1;
    case PKRRGPU_KKRR2: case PKRRGPU_BKRR2: return 2;
    default: return 3;
  }
}

int partitioner_of(int s) {
  switch (s) {
    case PKRRGPU_EXACT: return 0;
    case PKRRGPU_DCKRR: return 1;
    case PKRRGPU_KKRR: case PKRRGPU_KKRR2: case PKRRGPU_KKRR3: return 2;
    default: return 3;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// context: streams + caching device allocator
// ---------------------------------------------------------------------------
struct pkrrgpu_ctx {
  int device = 0;
  cudaStream_t main = nullptr;
  std::vector<cudaStream_t> work;      // graded priorities (highest first)
  std::vector<cudaStream_t> work_eq;   // equal (default) priority
  std::vector<cudaStream_t> aux, aux_eq;  // lookahead companions of work / work_eq (same priorities)
  cudaStream_t aux_main = nullptr;        // lookahead companion of main
  pk::Counter counter;
  double timings[8] = {0};
  std::vector<double> part_ms;  // last grid call: per-part Cholesky end, ms after the phase start
  std::vector<double> part_tl;  // last grid call, first cell: per part {gram0, gram1, chol0, chol1, pred1} ms after start
  // timing events of the grid calls: pooled (created once, re-recorded every call) and
  // turned into timings lazily -- at pkrrgpu_last_timings or the next call -- so a call
  // spends no host time on event creation / destruction / elapsed-time queries
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  struct Pending {
    bool on = false;
    cudaEvent_t all_a, all_b, part_a, part_b;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> gram, chol, pred;
    std::vector<cudaEvent_t> part_end;
    std::vector<std::array<cudaEvent_t, 5>> part_ev;
  } pending;
  cudaEvent_t pool_event() {
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      ck(cudaEventCreate(&e), "event");
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }
  void* pinned = nullptr;  // 64 KB pinned staging for small device->host reads
  double total_mem = 0.0;  // device HBM bytes
  std::multimap<size_t, void*> free_blocks;
  std::map<void*, size_t> live;
  size_t cached_bytes = 0;

  void* alloc(size_t bytes) {
    bytes = static_cast<size_t>(round_up(static_cast<int64_t>(bytes ? bytes : 256), 256));
    auto it = free_blocks.lower_bound(bytes);
    if (it != free_blocks.end() && it->first <= bytes * 2 + (1 << 20)) {
      void* p = it->second;
      live[p] = it->first;
      cached_bytes -= it->first;
      free_blocks.erase(it);
      return p;
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      trim();
      ck(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    live[p] = bytes;
    return p;
  }
  void release(void* p) {
    auto it = live.find(p);
    if (it == live.end()) return;
    free_blocks.emplace(it->second, p);
    cached_bytes += it->second;
    live.erase(it);
  }
  void trim() {
    cudaDeviceSynchronize();
    for (auto& kv : free_blocks) cudaFree(kv.second);
    free_blocks.clear();
    cached_bytes = 0;
  }
};

namespace {

// Per-call allocation scope: everything is returned to the cache at the end
// (after the context has synchronised its streams).
struct Scope {
  pkrrgpu_ctx* ctx;
  std::vector<void*> ptrs;
  explicit Scope(pkrrgpu_ctx* c) : ctx(c) {}
  ~Scope() {
    cudaDeviceSynchronize();
    for (void* p : ptrs) ctx->release(p);
    // bound the cache: a call that needed nearly all of HBM returns it, so other users
    // of the device can allocate; below that the blocks stay cached for the next call
    // (C4 holds ~0.8 of HBM: trimming it made every call re-allocate ~150 GB, ~0.2-0.5 s).
    // A later call that does not fit trims on cudaMalloc failure (pkrrgpu_ctx::alloc).
    if (static_cast<double>(ctx->cached_bytes) > 0.9 * ctx->total_mem) ctx->trim();
  }
  template <typename T>
  T* alloc(int64_t count) {
    void* p = ctx->alloc(sizeof(T) * static_cast<size_t>(count > 0 ? count : 1));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* zeros(int64_t count, cudaStream_t s) {
    T* p = alloc<T>(count);
    ck(cudaMemsetAsync(p, 0, sizeof(T) * static_cast<size_t>(count > 0 ? count : 1), s), "memset");
    return p;
  }
  // device view of a caller array (host or device pointer)
  template <typename T>
  const T* in(const T* src, int64_t count, cudaStream_t s) {
    if (!src || count <= 0) return src;
    if (is_device_ptr(src)) return src;
    T* p = alloc<T>(count);
    ck(cudaMemcpyAsync(p, src, sizeof(T) * count, cudaMemcpyHostToDevice, s), "H2D");
    return p;
  }
  template <typename T>
  T* upload(const std::vector<T>& v, cudaStream_t s) {
    T* p = alloc<T>(static_cast<int64_t>(v.size()));
    if (!v.empty())
      ck(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s), "H2D");
    return p;
  }
};

template <typename T>
void copy_out(T* dst, const T* dsrc, int64_t count, cudaStream_t s) {
  if (!dst || count <= 0) return;
  ck(cudaMemcpyAsync(dst, dsrc, sizeof(T) * count, cudaMemcpyDefault, s), "copy out");
}

template <typename T>
std::vector<T> to_host(const T* dsrc, int64_t count, cudaStream_t s) {
  std::vector<T> v(static_cast<size_t>(count > 0 ? count : 0));
  if (count > 0) {
    ck(cudaMemcpyAsync(v.data(), dsrc, sizeof(T) * count, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
  }
  return v;
}

// Result copies of a call batched through the context's pinned staging buffer: small
// device -> host copies become async copies into pinned memory plus one sync and host
// memcpys (a copy to pageable memory costs a synchronous staged transfer each); device
// destinations and large copies go direct.
struct D2HBatch {
  void* pinned;
  size_t cap;
  cudaStream_t s;
  struct Req {
    void* dst;
    const void* src;
    size_t bytes;
    size_t off;
  };
  std::vector<Req> staged;
  size_t used = 0;
  template <typename T>
  void add(T* dst, const T* src, int64_t count) {
    if (!dst || count <= 0) return;
    const size_t bytes = sizeof(T) * static_cast<size_t>(count);
    if (is_device_ptr(dst) || used + bytes > cap) {
      ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s), "copy out");
      return;
    }
    ck(cudaMemcpyAsync(static_cast<unsigned char*>(pinned) + used, src, bytes, cudaMemcpyDeviceToHost, s), "D2H");
    staged.push_back({dst, src, bytes, used});
    used = (used + bytes + 15) / 16 * 16;
  }
  void flush() {
    ck(cudaStreamSynchronize(s), "sync");
    for (const Req& r : staged) std::memcpy(r.dst, static_cast<unsigned char*>(pinned) + r.off, r.bytes);
    staged.clear();
    used = 0;
  }
};

__global__ void set_diag_kernel(double* A, int64_t from, int64_t mp, double v) {
  const int64_t i = from + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < mp) A[i * mp + i] = v;
}

__global__ void iota_kernel(int64_t* p, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = i;
}

__global__ void fill_i32_kernel(int32_t* p, int64_t n, int32_t v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void part_labels_kernel(const int64_t* order, const int64_t* bounds, int64_t p,
                                   int32_t* part_of, int64_t n) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= n) return;
  int64_t t = 0;
  while (t + 1 < p && bounds[t + 1] <= q) ++t;
  part_of[order[q]] = static_cast<int32_t>(t);
}

unsigned blocks_for(int64_t n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

// ---------------------------------------------------------------------------
// padded single-part buffers
// ---------------------------------------------------------------------------
struct PartBuf {
  int64_t m = 0, mp = 0, dp = 0;
  double* Xp = nullptr;     // mp x dp
  double* yp = nullptr;     // mp
  double* norms = nullptr;  // mp
  double* K = nullptr;      // mp x mp (full symmetric)
  double* A = nullptr;      // mp x mp (factor)
  double* Linv = nullptr;   // mp x 128
  double* z = nullptr;
  double* w = nullptr;      // fused forward-substitution accumulator (mp)
  double* alpha = nullptr;
  double* Ka = nullptr;
  bool assembled = false;   // A already holds K + lambda_0 m I (written by the gram's epilogue)
  int* scratch = nullptr;   // trsv tickets/flags
  int8_t* slices = nullptr; // Ozaki SYRK scratch: 2 x int8 [8 x mp x 512]
  int* exps = nullptr;      // [mp]
  CUtensorMap tmX, tmA, tmLinv;
};

void part_alloc(Scope& sc, PartBuf& pb, int64_t m, int64_t d, bool need_K, cudaStream_t s) {
  pb.m = m;
  pb.mp = round_up(m, kNB);
  pb.dp = round_up(d, 16);
  pb.Xp = sc.alloc<double>(pb.mp * pb.dp);
  pb.yp = sc.alloc<double>(pb.mp);
  pb.norms = sc.alloc<double>(pb.mp);
  if (need_K) pb.K = sc.alloc<double>(pb.mp * pb.mp);
  pb.A = sc.alloc<double>(pb.mp * pb.mp);
  pb.Linv = sc.zeros<double>(pb.mp * kNB, s);  // upper 32x32 blocks stay zero (the leaf writes lower)
  pb.z = sc.alloc<double>(pb.mp);
  pb.w = sc.alloc<double>(pb.mp);
  pb.alpha = sc.alloc<double>(pb.mp);
  pb.Ka = sc.alloc<double>(pb.mp * pk::kSymvSplit);
  pb.scratch = sc.alloc<int>(pk::trsv_scratch_ints(pb.mp));
  if (pk::syrk_ozaki()) {
    pb.slices = sc.alloc<int8_t>(2 * 8 * pb.mp * 512);  // two buffers: lookahead alternates them
    pb.exps = sc.alloc<int>(2 * pb.mp);
  }
  if (!pk::make_tmap(&pb.tmX, pb.Xp, pb.mp, pb.dp, pb.dp) ||
      !pk::make_tmap(&pb.tmA, pb.A, pb.mp, pb.mp, pb.mp) ||
      !pk::make_tmap(&pb.tmLinv, pb.Linv, pb.mp, kNB, kNB))
    fail(PKRRGPU_CUDA, "cuTensorMapEncodeTiled failed");
}

// Q rows (targets) padded to 64 for the cross-kernel tiles
struct QueryBuf {
  int64_t q = 0, qp = 0;
  double* Xq = nullptr;
  double* norms = nullptr;
  double* cross = nullptr;    // qp x mp (only the public cross-gram API materialises it)
  double* partial = nullptr;  // fused-prediction scratch (predict_partial_elems)
  double* pred = nullptr;     // qp
  CUtensorMap tmQ;
};

void query_alloc(Scope& sc, QueryBuf& qb, int64_t q, int64_t dp, int64_t mp, bool cross = false) {
  qb.q = q;
  qb.qp = round_up(q > 0 ? q : 1, 64);
  qb.Xq = sc.alloc<double>(qb.qp * dp);
  qb.norms = sc.alloc<double>(qb.qp);
  if (cross) qb.cross = sc.alloc<double>(qb.qp * mp);
  else qb.partial = sc.alloc<double>(pk::predict_partial_elems(qb.qp, mp));
  qb.pred = sc.alloc<double>(qb.qp);
  if (!pk::make_tmap(&qb.tmQ, qb.Xq, qb.qp, dp, dp)) fail(PKRRGPU_CUDA, "tensor map (Q)");
}

// ---------------------------------------------------------------------------
// clustering drivers (clustering.cpp:53-180)
// ---------------------------------------------------------------------------
struct ClusterOut {
  int32_t* label = nullptr;    // n
  double* centers = nullptr;   // k x d
  int64_t* sizes = nullptr;    // k (device)
  int64_t* start = nullptr;    // k
  int64_t* members = nullptr;  // n (row order within cluster)
  int64_t* tmp = nullptr;      // grouping scratch
  std::vector<int64_t> h_sizes, h_start;
  int iterations = 0;
};

void group_labels(pkrrgpu_ctx* ctx, Scope& sc, const int32_t* label, int64_t n, int k,
                  ClusterOut& co, cudaStream_t s) {
  if (!co.sizes) {
    co.sizes = sc.alloc<int64_t>(k);
    co.start = sc.alloc<int64_t>(k);
    co.members = sc.alloc<int64_t>(n);
    co.tmp = sc.alloc<int64_t>(((n + 255) / 256) * k + 2 * k);
  }
  pk::launch_group(label, n, k, co.sizes, co.start, co.members, co.tmp, s, ctx->counter);
}

// Sharded partition exchange (pkrrgpu_grid_args.allgather)
struct Exchange {
  pkrrgpu_allgather_fn fn = nullptr;
  void* user = nullptr;
  int rank = 0, world = 1;
  bool on() const { return fn != nullptr && world > 1; }
};

void exchange(pkrrgpu_ctx* ctx, const Exchange& ex, void* buf, int64_t bytes_per_rank) {
  ck(cudaStreamSynchronize(ctx->main), "sync");
  if (ex.fn(ex.user, buf, bytes_per_rank) != 0) fail(PKRRGPU_CUDA, "partition all-gather failed");
}

void kmeans_device(pkrrgpu_ctx* ctx, Scope& sc, const double* dX, int64_t n, int64_t d, int k,
                   uint64_t seed, double threshold, int max_iters, const double* xnorm,
                   ClusterOut& co, const Exchange* exg = nullptr) {
  cudaStream_t s = ctx->main;
  if (k < 1 || static_cast<int64_t>(k) > n) fail(PKRRGPU_INVALID, "kmeans: need 1 <= k <= n");
  // Sharded (one process per GPU): rank r assigns rows [r S, (r+1) S) and updates
  // clusters [r Kc, (r+1) Kc); labels and centres are all-gathered each iteration, the
  // changed count is recounted globally.  Each row's argmin and each cluster's
  // sequential chain is the single-process computation: bitwise the same result.
  const Exchange ex = exg ? *exg : Exchange{};
  const bool shard = ex.on();
  const int W = shard ? ex.world : 1, R = shard ? ex.rank : 0;
  const int64_t S = (n + W - 1) / W;
  const int Kc = (k + W - 1) / W;
  const int64_t r0 = std::min<int64_t>(n, R * S), r1 = std::min<int64_t>(n, (R + 1) * S);
  const int j0 = std::min(k, R * Kc), j1 = std::min(k, (R + 1) * Kc);
  co.label = sc.alloc<int32_t>(W * S);
  co.centers = sc.alloc<double>(static_cast<int64_t>(W) * Kc * d);
  // init: k distinct samples, Rng(seed) + random_permutation (clustering.cpp:64-68)
  HostRng rng(seed);
  const std::vector<int64_t> perm = rng.permutation(n);
  std::vector<int64_t> first(perm.begin(), perm.begin() + k);
  int64_t* didx = sc.upload(first, s);
  pk::launch_gather_rows(dX, d, didx, k, co.centers, k, d, s, ctx->counter);
  fill_i32_kernel<<<blocks_for(n), 256, 0, s>>>(co.label, n, -1);
  ctx->counter.launched();
  double* best = sc.alloc<double>(W * S);
  double* cnorm = sc.alloc<double>(k);
  int32_t* prev = shard ? sc.alloc<int32_t>(n) : nullptr;
  unsigned long long* changed = sc.alloc<unsigned long long>(2);
  unsigned long long* far = sc.alloc<unsigned long long>(2);
  std::vector<int64_t> sz(k);
  cudaEvent_t ev_sizes;
  ck(cudaEventCreateWithFlags(&ev_sizes, cudaEventDisableTiming), "event");
  auto update = [&]() {  // centroid update of this rank's clusters, then the exchange
    pk::launch_means(dX, d, co.members, co.start, co.sizes, k, co.centers, s, ctx->counter, j0, j1);
  };
  int iter = 0;
  for (; iter < max_iters; ++iter) {
    pk::launch_row_norms(co.centers, k, d, d, cnorm, s, ctx->counter);
    ck(cudaMemsetAsync(changed, 0, sizeof(unsigned long long), s), "memset");
    if (shard) ck(cudaMemcpyAsync(prev, co.label, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s), "copy");
    pk::launch_assign(dX, r1, d, xnorm, co.centers, cnorm, k, 0, nullptr, r0, co.label, best, changed, s,
                      ctx->counter);
    if (shard) {
      exchange(ctx, ex, co.label, S * static_cast<int64_t>(sizeof(int32_t)));
      pk::launch_label_diff(prev, co.label, n, changed, s, ctx->counter);
    }
    group_labels(ctx, sc, co.label, n, k, co, s);
    // one round trip per iteration: sizes and the changed count together.  The centroid
    // update is enqueued before the host looks at them (speculatively: it only has to
    // be redone when a cluster is empty and gets reseeded below), so the host decision
    // overlaps the update instead of idling the GPU
    {
      auto* pin = static_cast<unsigned char*>(ctx->pinned);
      ck(cudaMemcpyAsync(pin, co.sizes, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaMemcpyAsync(pin + sizeof(int64_t) * k, changed, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                         s),
         "D2H");
      ck(cudaEventRecord(ev_sizes, s), "event");
      update();
      ck(cudaEventSynchronize(ev_sizes), "sync");
      std::memcpy(sz.data(), pin, sizeof(int64_t) * k);
    }
    unsigned long long ch = 0;
    std::memcpy(&ch, static_cast<unsigned char*>(ctx->pinned) + sizeof(int64_t) * k, sizeof(ch));
    // empty-cluster reseed (clustering.cpp:98-117)
    bool reseeded = false;
    for (int j = 0; j < k; ++j) {
      if (sz[j] != 0) continue;
      if (shard && !reseeded) exchange(ctx, ex, best, S * static_cast<int64_t>(sizeof(double)));
      ck(cudaMemcpyAsync(co.sizes, sz.data(), sizeof(int64_t) * k, cudaMemcpyHostToDevice, s), "H2D");
      pk::launch_farthest(best, co.label, co.sizes, n, far, s, ctx->counter);
      const std::vector<unsigned long long> f = to_host(far, 2, s);
      const int64_t far_i = f[0] == 0 ? 0 : static_cast<int64_t>(f[1]);
      int32_t old = to_host(co.label + far_i, 1, s)[0];
      --sz[old];
      const int32_t jj = j;
      const double zero = 0.0;
      ck(cudaMemcpyAsync(co.label + far_i, &jj, sizeof(int32_t), cudaMemcpyHostToDevice, s), "H2D");
      ck(cudaMemcpyAsync(best + far_i, &zero, sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
      ck(cudaStreamSynchronize(s), "sync");
      sz[j] = 1;
      ++ch;
      reseeded = true;
    }
    if (reseeded) {  // the speculative update saw an empty cluster: regroup and redo it
      group_labels(ctx, sc, co.label, n, k, co, s);
      update();
    }
    if (shard) exchange(ctx, ex, co.centers, static_cast<int64_t>(Kc) * d * static_cast<int64_t>(sizeof(double)));
    if (static_cast<double>(ch) / static_cast<double>(n) <= threshold) {
      ++iter;
      break;
    }
  }
  cudaEventDestroy(ev_sizes);
  co.iterations = iter;
  co.h_sizes = to_host(co.sizes, k, s);
  co.h_start = to_host(co.start, k, s);
}

void kbalance_device(pkrrgpu_ctx* ctx, Scope& sc, const double* dX, int64_t n, int64_t d, int k,
                     uint64_t seed, double threshold, int max_iters, bool recompute,
                     const double* xnorm, ClusterOut& co, const Exchange* ex = nullptr) {
  if (k < 1 || static_cast<int64_t>(k) > n) fail(PKRRGPU_INVALID, "kbalance: need 1 <= k <= n");
  kmeans_device(ctx, sc, dX, n, d, k, seed, threshold, max_iters, xnorm, co, ex);  // the warm start
  cudaStream_t s = ctx->main;
  const int64_t base = n / k, extra = n % k;
  // exact parallel replay of the sequential capacity scan (clustering.cpp:159-176):
  // between two closure events every remaining sample's choice is the argmin over
  // a fixed open set; the next event is the first position where some open
  // cluster reaches its cap.  <= k+1 rounds.
  fill_i32_kernel<<<blocks_for(n), 256, 0, s>>>(co.label, n, -1);
  ctx->counter.launched();
  double* cnorm = sc.alloc<double>(k);
  pk::launch_row_norms(co.centers, k, d, d, cnorm, s, ctx->counter);
  std::vector<int64_t> sizes(k, 0), thr(k);
  std::vector<uint8_t> open(k, 1);
  uint8_t* dopen = sc.alloc<uint8_t>(k);
  int64_t* dthr = sc.alloc<int64_t>(k);
  int64_t* dpos = sc.alloc<int64_t>(k);
  int64_t* dhist = sc.alloc<int64_t>(k);
  int64_t grown = 0, pos = 0;
  while (pos < n) {
    ck(cudaMemcpyAsync(dopen, open.data(), k, cudaMemcpyHostToDevice, s), "H2D");
    pk::launch_assign(dX, n, d, xnorm, co.centers, cnorm, k, 1, dopen, pos, co.label, nullptr, nullptr,
                      s, ctx->counter);
    for (int j = 0; j < k; ++j)
      thr[j] = open[j] ? (grown < extra ? base + 1 - sizes[j] : base - sizes[j]) : 0;
    ck(cudaMemcpyAsync(dthr, thr.data(), sizeof(int64_t) * k, cudaMemcpyHostToDevice, s), "H2D");
    pk::launch_events(co.label, pos, n, k, dthr, dpos, s, ctx->counter);
    const std::vector<int64_t> ev = to_host(dpos, k, s);
    int64_t e = INT64_MAX;
    int jstar = -1;
    for (int j = 0; j < k; ++j)
      if (ev[j] < e) {
        e = ev[j];
        jstar = j;
      }
    const int64_t last = jstar < 0 ? n - 1 : e;
    pk::launch_hist(co.label, pos, last, k, dhist, s, ctx->counter);
    const std::vector<int64_t> h = to_host(dhist, k, s);
    int64_t added = 0;
    for (int j = 0; j < k; ++j) {
      sizes[j] += h[j];
      added += h[j];
    }
    if (added != last - pos + 1) fail(PKRRGPU_LOGIC, "kbalance: no open cluster");
    if (jstar < 0) break;
    if (grown < extra) {
      ++grown;  // jstar grew to base + 1
      open[jstar] = 0;
      if (grown == extra)
        for (int j = 0; j < k; ++j)
          if (sizes[j] == base) open[j] = 0;
    } else {
      open[jstar] = 0;  // reached base with no growth slots left
    }
    pos = e + 1;
  }
  group_labels(ctx, sc, co.label, n, k, co, s);
  if (recompute) pk::launch_means(dX, d, co.members, co.start, co.sizes, k, co.centers, s, ctx->counter);
  co.h_sizes = to_host(co.sizes, k, s);
  co.h_start = to_host(co.start, k, s);
}

// make_partition (strategies.cpp:64-102) on device.  Returns p_eff.
struct PartitionOut {
  int64_t p = 0;
  int32_t* part_of = nullptr;   // n
  int64_t* order = nullptr;     // n (rows part by part)
  double* centers = nullptr;    // p x d or null
  std::vector<int64_t> sizes, start;
  int iterations = 0;
};

void make_partition_device(pkrrgpu_ctx* ctx, Scope& sc, int strategy, const double* dX, int64_t n,
                           int64_t d, int64_t p, uint64_t seed, double thr, int max_iters,
                           PartitionOut& po, const Exchange* ex = nullptr) {
  cudaStream_t s = ctx->main;
  const int pk_kind = partitioner_of(strategy);
  if (pk_kind == 0) {
    po.p = 1;
    po.part_of = sc.zeros<int32_t>(n, s);
    po.order = sc.alloc<int64_t>(n);
    iota_kernel<<<blocks_for(n), 256, 0, s>>>(po.order, n);
    ctx->counter.launched();
    po.sizes = {n};
    po.start = {0};
    return;
  }
  if (p < 1 || p > n) fail(PKRRGPU_INVALID, "partition: need 1 <= p <= n");
  po.p = p;
  if (pk_kind == 1) {
    HostRng rng(seed);
    const std::vector<int64_t> perm = rng.permutation(n);
    po.order = sc.upload(perm, s);
    const int64_t base = n / p, extra = n % p;
    std::vector<int64_t> bounds(p + 1, 0);
    po.sizes.resize(p);
    po.start.resize(p);
    for (int64_t t = 0; t < p; ++t) {
      po.sizes[t] = base + (t < extra ? 1 : 0);
      po.start[t] = bounds[t];
      bounds[t + 1] = bounds[t] + po.sizes[t];
    }
    int64_t* db = sc.upload(bounds, s);
    po.part_of = sc.alloc<int32_t>(n);
    part_labels_kernel<<<blocks_for(n), 256, 0, s>>>(po.order, db, p, po.part_of, n);
    ctx->counter.launched();
    return;
  }
  double* xnorm = sc.alloc<double>(n);
  pk::launch_row_norms(dX, n, d, d, xnorm, s, ctx->counter);
  ClusterOut co;
  if (pk_kind == 2)
    kmeans_device(ctx, sc, dX, n, d, static_cast<int>(p), seed, thr, max_iters, xnorm, co, ex);
  else
    kbalance_device(ctx, sc, dX, n, d, static_cast<int>(p), seed, thr, max_iters, true, xnorm, co, ex);
  po.part_of = co.label;
  po.order = co.members;
  po.centers = co.centers;
  po.sizes = co.h_sizes;
  po.start = co.h_start;
  po.iterations = co.iterations;
}

// nearest_center routing of q rows (clustering.cpp:182-195) + stable grouping
struct RouteOut {
  int32_t* route = nullptr;
  int64_t* members = nullptr;
  std::vector<int64_t> sizes, start;
};

void route_rows(pkrrgpu_ctx* ctx, Scope& sc, const double* dQ, int64_t q, int64_t d,
                const double* centers, int k, RouteOut& ro) {
  cudaStream_t s = ctx->main;
  double* qn = sc.alloc<double>(q);
  double* cn = sc.alloc<double>(k);
  pk::launch_row_norms(dQ, q, d, d, qn, s, ctx->counter);
  pk::launch_row_norms(centers, k, d, d, cn, s, ctx->counter);
  ro.route = sc.alloc<int32_t>(q);
  fill_i32_kernel<<<blocks_for(q), 256, 0, s>>>(ro.route, q, -1);
  ctx->counter.launched();
  pk::launch_assign(dQ, q, d, qn, centers, cn, k, 0, nullptr, 0, ro.route, nullptr, nullptr, s,
                    ctx->counter);
  ClusterOut co;
  group_labels(ctx, sc, ro.route, q, k, co, s);
  ro.members = co.members;
  ro.sizes = to_host(co.sizes, k, s);
  ro.start = to_host(co.start, k, s);
}

// ---------------------------------------------------------------------------
// one part: gram -> assemble -> potrf -> solve -> residual (train_krr)
// ---------------------------------------------------------------------------
void part_load(pkrrgpu_ctx* ctx, PartBuf& pb, const double* dX, const double* dy, int64_t d,
               const int64_t* rows, cudaStream_t s) {
  pk::launch_gather_rows(dX, d, rows, pb.m, pb.Xp, pb.mp, pb.dp, s, ctx->counter);
  pk::launch_gather_vec(dy, rows, pb.m, pb.yp, pb.mp, s, ctx->counter);
  pk::launch_row_norms(pb.Xp, pb.mp, pb.dp, pb.dp, pb.norms, s, ctx->counter);
}

void part_solve(pkrrgpu_ctx* ctx, PartBuf& pb, double lambda, int* status, double* res_out,
                cudaStream_t s, cudaStream_t s2, bool alone, bool assembled = false) {
  const double shift = lambda * static_cast<double>(pb.m);
  if (!assembled) pk::launch_assemble(pb.K, pb.A, pb.mp, shift, status, s, ctx->counter, /*lower_only=*/true);
  const pk::FwdSolve fs{pb.yp, pb.w, pb.z};
  if (pk::launch_potrf(pb.A, pb.tmA, pb.tmLinv, pb.Linv, pb.mp, pb.m, status, s, ctx->counter, pb.slices,
                       pb.exps, s2, alone, &fs))
    pk::launch_trsv_bwd(pb.A, pb.Linv, pb.mp, pb.z, pb.alpha, pb.scratch, status, s, ctx->counter);
  else
    pk::launch_trsv(pb.A, pb.Linv, pb.mp, pb.yp, pb.z, pb.alpha, pb.scratch, status, s, ctx->counter);
  if (res_out) {
    pk::launch_symv_lower(pb.K, pb.mp, pb.alpha, pb.Ka, status, s, ctx->counter);
    pk::launch_residual_finish(pb.Ka, pb.alpha, pb.yp, pb.m, shift, res_out, status, s, ctx->counter);
  }
}

struct Timer {
  cudaEvent_t a, b;
  Timer() {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

bool df_gram_fused() {
  static const bool on = std::getenv("PKRR_DF_GRAM") && std::atoi(std::getenv("PKRR_DF_GRAM")) != 0;
  return on;
}

double chol_flops(int64_t m) {
  const double mu = static_cast<double>(m);
  return mu * (mu + 1) * (2 * mu + 1) / 6.0;
}

// Cell combine + reference-order MSE + best cell (strategies.cpp:458-505) on device:
// pred [ncell x P x t]; failed cells get NaN and never win; best = first strict
// minimum in trace order.  Returns the best index (-1 when every cell failed) and
// copies its combined prediction to best_pred (host or device, may be null).
int64_t combine_cells(pkrrgpu_ctx* ctx, Scope& sc, int predictor, int64_t P, int64_t t, int64_t ncell,
                      const double* pred, const double* y, const std::vector<uint8_t>& cfail,
                      std::vector<double>& cmse, double* best_pred) {
  cudaStream_t s = ctx->main;
  double* comb = sc.alloc<double>(ncell * t);
  double* dm = sc.alloc<double>(ncell);
  pk::launch_combine_cells(pred, P, t, ncell, predictor, y, comb, dm, s, ctx->counter);
  cmse = to_host(dm, ncell, s);
  int64_t best = -1;
  for (int64_t c = 0; c < ncell; ++c) {
    if (cfail[c]) {
      cmse[c] = std::numeric_limits<double>::quiet_NaN();
      continue;
    }
    if (best < 0 || cmse[c] < cmse[best]) best = c;
  }
  if (best >= 0 && best_pred) copy_out(best_pred, comb + best * t, t, s);
  return best;
}

int guard(pkrrgpu_ctx* ctx) {
  if (!ctx) {
    g_err = "null context";
    return PKRRGPU_INVALID;
  }
  ck(cudaSetDevice(ctx->device), "cudaSetDevice");
  ctx->counter.reset();
  return 0;
}

// Every kernel launch of the call was checked (pk::Counter::launched): a failed launch
// turns the call's status into PKRRGPU_CUDA even though later work was enqueued.
int launch_status(pkrrgpu_ctx* ctx) {
  if (ctx->counter.err == cudaSuccess) return PKRRGPU_OK;
  g_err = std::string("kernel launch failed (launch #") + std::to_string(ctx->counter.err_at) +
          "): " + cudaGetErrorString(ctx->counter.err);
  return PKRRGPU_CUDA;
}

}  // namespace

#define API_BEGIN \
  try {           \
    if (int g_ = guard(ctx)) return g_;
#define API_RETURN_OK return launch_status(ctx)
#define API_END                                      \
  return launch_status(ctx);                         \
  }                                                  \
  catch (const Fail& f) {                            \
    return f.code;                                   \
  }                                                  \
  catch (const std::exception& e) {                  \
    g_err = e.what();                                \
    return PKRRGPU_CUDA;                             \
  }

extern "C" {

const char* pkrrgpu_version(void) { return "pkrr-b200 0.1 (sm_100a, DMMA f64 + TMA)"; }
const char* pkrrgpu_last_error(void) { return g_err.c_str(); }
// internal (multi.cu): a worker thread's error reported on the calling thread
void pkrrgpu_set_last_error_(const char* msg) { g_err = msg ? msg : ""; }
// internal (dist.cu)
int pkrrgpu_context_device_(const pkrrgpu_ctx* ctx) { return ctx ? ctx->device : 0; }
// internal (dist.cu): launches made on a context's device outside its own calls
void pkrrgpu_add_launches_(pkrrgpu_ctx* ctx, int64_t n) {
  if (ctx) ctx->counter.launches += n;
}

int pkrrgpu_create(int device, pkrrgpu_ctx** out) {
  try {
    if (!out) fail(PKRRGPU_INVALID, "null out");
    // The grid runs up to 17 streams (8 part streams, their 8 lookahead companions,
    // main); with the default 8 hardware work queues streams share queues and pick up
    // false dependencies.  Read at context creation: effective when this library
    // creates the context (the Python package sets it at import as well).
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) fail(PKRRGPU_INVALID, "no such CUDA device");
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "props");
    if (prop.major != 10) fail(PKRRGPU_CUDA, "pkrr-b200 needs an sm_100a (Blackwell) device");
    const double total_mem = static_cast<double>(prop.totalGlobalMem);
    auto* c = new pkrrgpu_ctx();
    c->device = device;
    c->total_mem = total_mem;
    if (const char* f = std::getenv("PKRR_FAULT_LAUNCH")) c->counter.fault_at = std::atoll(f);
    if (const char* g = std::getenv("PKRR_PANEL_GROUP")) pk::set_panel_group(std::atoi(g));
    if (const char* g = std::getenv("PKRR_SYRK_PERSISTENT")) pk::set_syrk_persistent(std::atoi(g));
    if (const char* g = std::getenv("PKRR_SYRK")) pk::set_syrk_ozaki(std::strcmp(g, "ozaki") == 0 ? 1 : 0);
    int least = 0, greatest = 0;
    ck(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
    // the panel chain of a factorisation outranks its lookahead trailing update
    ck(cudaStreamCreateWithPriority(&c->main, cudaStreamNonBlocking, greatest), "stream");
    ck(cudaMallocHost(&c->pinned, 64 * 1024), "pinned");
    // work streams in decreasing priority: the grid maps parts to them largest
    // first (LPT on one GPU), so the critical part wins the block scheduler
    c->work.resize(8);
    c->work_eq.resize(8);
    c->aux.resize(8);
    c->aux_eq.resize(8);
    for (size_t i = 0; i < c->work.size(); ++i) {
      int prio = greatest + static_cast<int>(i);
      if (prio > least) prio = least;
      const int below = prio + 1 > least ? least : prio + 1;
      const int eq = least - 1 < greatest ? greatest : least - 1;
      ck(cudaStreamCreateWithPriority(&c->work[i], cudaStreamNonBlocking, prio), "stream");
      ck(cudaStreamCreateWithPriority(&c->work_eq[i], cudaStreamNonBlocking, eq), "stream");
      ck(cudaStreamCreateWithPriority(&c->aux[i], cudaStreamNonBlocking, below), "stream");
      ck(cudaStreamCreateWithPriority(&c->aux_eq[i], cudaStreamNonBlocking, least), "stream");
    }
    ck(cudaStreamCreateWithPriority(&c->aux_main, cudaStreamNonBlocking, least), "stream");
    *out = c;
    return PKRRGPU_OK;
  } catch (const Fail& f) {
    return f.code;
  }
}

void pkrrgpu_destroy(pkrrgpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  ctx->trim();
  for (auto& kv : ctx->live) cudaFree(kv.first);
  for (auto s : ctx->work) cudaStreamDestroy(s);
  for (auto s : ctx->work_eq) cudaStreamDestroy(s);
  for (auto s : ctx->aux) cudaStreamDestroy(s);
  for (auto s : ctx->aux_eq) cudaStreamDestroy(s);
  if (ctx->aux_main) cudaStreamDestroy(ctx->aux_main);
  cudaStreamDestroy(ctx->main);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  delete ctx;
}

int pkrrgpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int64_t pkrrgpu_launch_count(const pkrrgpu_ctx* ctx) { return ctx ? ctx->counter.launches : 0; }

void* pkrrgpu_stream(pkrrgpu_ctx* ctx) { return ctx ? static_cast<void*>(ctx->main) : nullptr; }

int pkrrgpu_wait_stream(pkrrgpu_ctx* ctx, void* stream) {
  API_BEGIN
  cudaEvent_t e;
  ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  ck(cudaEventRecord(e, static_cast<cudaStream_t>(stream)), "event");
  ck(cudaStreamWaitEvent(ctx->main, e, 0), "wait");
  ck(cudaEventDestroy(e), "event");
  API_END
}

int pkrrgpu_probe_potrf(pkrrgpu_ctx* ctx, int64_t m, int alone, double* out) {
  API_BEGIN
  if (m <= 0 || !out) fail(PKRRGPU_INVALID, "probe_potrf: bad arguments");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  // SPD test system: gaussian gram of m seeded points (d = 90) + 1e-4 * m * I
  const int64_t d = 90;
  std::vector<double> X(m * d);
  std::mt19937_64 eng(12345);
  std::normal_distribution<double> nd(0.0, 1.0);
  for (auto& v : X) v = nd(eng);
  PartBuf pb;
  part_alloc(sc, pb, m, d, true, s);
  const double* dX = sc.in(X.data(), m * d, s);
  int64_t* idx = sc.alloc<int64_t>(m);
  iota_kernel<<<blocks_for(m), 256, 0, s>>>(idx, m);
  ctx->counter.launched();
  pk::launch_gather_rows(dX, d, idx, m, pb.Xp, pb.mp, pb.dp, s, ctx->counter);
  pk::launch_row_norms(pb.Xp, pb.mp, pb.dp, pb.dp, pb.norms, s, ctx->counter);
  pk::launch_gram_sym(pb.tmX, pb.norms, pb.mp, pb.dp, m, 3.0, pb.K, pb.mp, nullptr, s, ctx->counter, false);
  int* status = sc.zeros<int>(2, s);
  pk::launch_assemble(pb.K, pb.A, pb.mp, 1e-4 * static_cast<double>(m), status, s, ctx->counter, true);
  ck(cudaStreamSynchronize(s), "sync");
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  std::vector<double> fl;
  Timer tm;
  pk::set_syrk_probe(&ev, &fl);
  ck(cudaEventRecord(tm.a, s), "event");
  pk::launch_potrf(pb.A, pb.tmA, pb.tmLinv, pb.Linv, pb.mp, m, status, s, ctx->counter, pb.slices, pb.exps,
                   nullptr, alone != 0);
  ck(cudaEventRecord(tm.b, s), "event");
  pk::set_syrk_probe(nullptr, nullptr);
  ck(cudaStreamSynchronize(s), "sync");
  float total = 0;
  cudaEventElapsedTime(&total, tm.a, tm.b);
  double syrk_ms = 0, syrk_fl = 0;
  for (size_t i = 0; i < ev.size(); ++i) {
    float msi = 0;
    cudaEventElapsedTime(&msi, ev[i].first, ev[i].second);
    syrk_ms += msi;
    syrk_fl += fl[i];
    cudaEventDestroy(ev[i].first);
    cudaEventDestroy(ev[i].second);
  }
  out[0] = total;                      // whole factorization, ms
  out[1] = chol_flops(m);              // its algorithmic flops
  out[2] = syrk_ms;                    // trailing-SYRK launches, ms (sum)
  out[3] = syrk_fl;                    // their algorithmic flops
  out[4] = static_cast<double>(ev.size());
  out[5] = to_host(status, 1, s)[0];   // NPD flag (must be 0)
  API_END
}

int pkrrgpu_fp64_peak(pkrrgpu_ctx* ctx, double* tflops) {
  API_BEGIN
  if (!tflops) fail(PKRRGPU_INVALID, "null out");
  int sms = 0;
  ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device), "attr");
  double* sink = nullptr;
  ck(cudaMalloc(&sink, 4096), "malloc");
  Timer tm;
  const int blocks = sms * 2, threads = 512, iters = 20000;
  pk::launch_dmma_probe(blocks, threads, 200, sink, ctx->main, ctx->counter);
  ck(cudaEventRecord(tm.a, ctx->main), "event");
  pk::launch_dmma_probe(blocks, threads, iters, sink, ctx->main, ctx->counter);
  ck(cudaEventRecord(tm.b, ctx->main), "event");
  ck(cudaEventSynchronize(tm.b), "sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, tm.a, tm.b);
  cudaFree(sink);
  *tflops = 2.0 * 256.0 * 8.0 * iters * blocks * (threads / 32) / (ms * 1e-3) / 1e12;
  API_END
}

namespace {
// the last grid call's phase timings from its (completed) pooled events
void finalize_timings(pkrrgpu_ctx* ctx) {
  pkrrgpu_ctx::Pending& P = ctx->pending;
  if (!P.on) return;
  P.on = false;
  // union of [start, end] intervals (ms after the call start)
  auto union_ms = [&](const std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& iv) {
    std::vector<std::pair<float, float>> x;
    for (const auto& v : iv) {
      float a0 = 0, a1 = 0;
      cudaEventElapsedTime(&a0, P.all_a, v.first);
      cudaEventElapsedTime(&a1, P.all_a, v.second);
      x.push_back({a0, a1});
    }
    std::sort(x.begin(), x.end());
    double tot = 0, cs = -1, ce = -1;
    for (auto& v : x) {
      if (v.first > ce) {
        if (ce > cs) tot += ce - cs;
        cs = v.first;
        ce = v.second;
      } else if (v.second > ce) {
        ce = v.second;
      }
    }
    if (ce > cs) tot += ce - cs;
    return tot;
  };
  const double ms_gram = union_ms(P.gram), ms_chol = union_ms(P.chol), ms_pred = union_ms(P.pred);
  float chol0 = 1e30f;
  for (const auto& v : P.chol) {
    float a0 = 0;
    cudaEventElapsedTime(&a0, P.all_a, v.first);
    chol0 = std::min(chol0, a0);
  }
  float ms_part = 0, ms_all = 0;
  cudaEventElapsedTime(&ms_part, P.part_a, P.part_b);
  cudaEventElapsedTime(&ms_all, P.all_a, P.all_b);
  ctx->timings[0] = ms_part;
  ctx->timings[1] = ms_all - ms_part;
  ctx->timings[2] = ms_pred;
  ctx->timings[3] = ms_all;
  ctx->timings[4] = ms_chol;
  ctx->timings[5] = ms_gram;
  const size_t p = P.part_end.size();
  ctx->part_ms.assign(p, 0.0);
  for (size_t q = 0; q < p; ++q)
    if (P.part_end[q]) {
      float ms = 0;
      cudaEventElapsedTime(&ms, P.all_a, P.part_end[q]);
      ctx->part_ms[q] = ms - chol0;
    }
  ctx->part_tl.assign(5 * p, 0.0);
  for (size_t q = 0; q < p; ++q)
    for (int j = 0; j < 5; ++j)
      if (P.part_ev[q][j]) {
        float ms = 0;
        cudaEventElapsedTime(&ms, P.all_a, P.part_ev[q][j]);
        ctx->part_tl[5 * q + j] = ms;
      }
  cudaGetLastError();
}
}  // namespace

int pkrrgpu_last_timings(const pkrrgpu_ctx* cctx, double* ms, int n) {
  if (!cctx || !ms) return PKRRGPU_INVALID;
  pkrrgpu_ctx* ctx = const_cast<pkrrgpu_ctx*>(cctx);
  if (ctx->pending.on) {
    cudaSetDevice(ctx->device);
    finalize_timings(ctx);
  }
  for (int i = 0; i < n && i < 8; ++i) ms[i] = ctx->timings[i];
  // [8 ...]: per-part Cholesky completion (ms after the first Cholesky phase start)
  const int np = static_cast<int>(ctx->part_ms.size());
  for (int i = 8; i < n && i - 8 < np; ++i) ms[i] = ctx->part_ms[i - 8];
  // [8 + p ...]: per part {gram start, gram end, Cholesky start, Cholesky end, predict end}
  // of the first cell, ms after the grid call's start event
  for (int i = 8 + np; i < n && i - 8 - np < static_cast<int>(ctx->part_tl.size()); ++i)
    ms[i] = ctx->part_tl[i - 8 - np];
  return PKRRGPU_OK;
}

// ---- data preparation ---------------------------------------------------------
namespace {
// rng.cpp:36-56: sub_seed = splitmix64(splitmix64(seed ^ fnv1a64(tag)))
uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
uint64_t fnv1a64(const char* s) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (; *s; ++s) {
    h ^= static_cast<unsigned char>(*s);
    h *= 0x100000001B3ull;
  }
  return h;
}
uint64_t sub_seed(uint64_t seed, const char* tag) { return splitmix64(splitmix64(seed ^ fnv1a64(tag))); }
}  // namespace

int pkrrgpu_standardize(pkrrgpu_ctx* ctx, const double* X_train, int64_t n, int64_t d, const double* X_test,
                        int64_t t, double* train_out, double* test_out, double* mean_out, double* stddev_out) {
  API_BEGIN
  if (n <= 0) fail(PKRRGPU_INVALID, "standardize: empty training set");
  if (d <= 0 || !X_train || !train_out) fail(PKRRGPU_INVALID, "standardize: null input");
  if (t > 0 && (!X_test || !test_out)) fail(PKRRGPU_INVALID, "standardize: null test input");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dX = sc.in(X_train, n * d, s);
  double* mean = sc.alloc<double>(d);
  double* sd = sc.alloc<double>(d);
  if (!pk::launch_standardize_stats(dX, n, d, d, mean, sd, s, ctx->counter)) {
    // odd d or unaligned caller pointer: stream a copy with an even (16-byte) row pitch
    const int64_t ld = round_up(d, 2);
    double* P = sc.alloc<double>(n * ld);
    ck(cudaMemcpy2DAsync(P, sizeof(double) * ld, dX, sizeof(double) * d, sizeof(double) * d, n,
                         cudaMemcpyDeviceToDevice, s),
       "pitch copy");
    if (!pk::launch_standardize_stats(P, n, d, ld, mean, sd, s, ctx->counter))
      fail(PKRRGPU_CUDA, "standardize: tensor map");
  }
  double* out = is_device_ptr(train_out) ? train_out : sc.alloc<double>(n * d);
  pk::launch_standardize_apply(dX, n, d, mean, sd, out, s, ctx->counter);
  copy_out(train_out, static_cast<const double*>(out), out == train_out ? 0 : n * d, s);
  if (t > 0) {
    const double* dT = sc.in(X_test, t * d, s);
    double* tout = is_device_ptr(test_out) ? test_out : sc.alloc<double>(t * d);
    pk::launch_standardize_apply(dT, t, d, mean, sd, tout, s, ctx->counter);
    copy_out(test_out, static_cast<const double*>(tout), tout == test_out ? 0 : t * d, s);
  }
  copy_out(mean_out, static_cast<const double*>(mean), d, s);
  copy_out(stddev_out, static_cast<const double*>(sd), d, s);
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

int pkrrgpu_auto_sigma_grid(pkrrgpu_ctx* ctx, const double* X, int64_t n, int64_t d, uint64_t seed,
                            double* grid_out) {
  API_BEGIN
  if (!grid_out || (n > 0 && (!X || d <= 0))) fail(PKRRGPU_INVALID, "auto_sigma_grid: null argument");
  const int64_t cnt = n < 512 ? n : 512;
  double g = 1.0;
  if (cnt > 1) {
    Scope sc(ctx);
    cudaStream_t s = ctx->main;
    HostRng rng(sub_seed(seed, "sigma-grid"));
    std::vector<int64_t> perm = rng.permutation(n);
    perm.resize(cnt);
    const double* dX = sc.in(X, n * d, s);
    int64_t* didx = sc.upload(perm, s);
    double* G = sc.alloc<double>(cnt * d);
    double* nrm = sc.alloc<double>(cnt);
    pk::launch_gather_rows(dX, d, didx, cnt, G, cnt, d, s, ctx->counter);
    pk::launch_row_norms(G, cnt, d, d, nrm, s, ctx->counter);
    const int64_t np = cnt * (cnt - 1) / 2;
    double* dist = sc.alloc<double>(np);
    pk::launch_pair_dist(G, nrm, cnt, d, dist, s, ctx->counter);
    std::vector<double> h = to_host(dist, np, s);
    // lower median of the sorted distances (strategies.cpp:224-229): any selection
    // of the ((np - 1) / 2)-th smallest value gives the same number
    std::nth_element(h.begin(), h.begin() + (np - 1) / 2, h.end());
    const double median = h[(np - 1) / 2];
    if (median > 0.0) g = median;
  }
  for (int e = -4; e <= 4; ++e) grid_out[e + 4] = g * std::ldexp(1.0, e);
  API_END
}

// ---- LIBSVM loader (dataset.cpp:83-125) ------------------------------------------
struct pkrrgpu_dataset {
  int64_t n = 0, d = 0;
  std::vector<int64_t> row_ptr{0};
  std::vector<int32_t> col;
  std::vector<double> val;
  std::vector<double> y;
  double* pinned = nullptr;  // dense staging (n x d), cudaMallocHost
  ~pkrrgpu_dataset() {
    if (pinned) cudaFreeHost(pinned);
  }
};

namespace {
struct LibsvmChunk {
  std::vector<int64_t> row_nnz;
  std::vector<int32_t> col;
  std::vector<double> val, y;
  int64_t max_col = -1;
  int64_t err_line = -1;  // first failing line (1-based) in this chunk
  std::string err;
};

// parse lines [b, e) of the buffer; line numbers start at first_line
void parse_libsvm_lines(const char* buf, const std::vector<int64_t>& starts, int64_t b, int64_t e,
                        int64_t total_len, LibsvmChunk& out) {
  std::string line;
  for (int64_t li = b; li < e; ++li) {
    const int64_t s0 = starts[li];
    int64_t s1 = li + 1 < static_cast<int64_t>(starts.size()) ? starts[li + 1] - 1 : total_len;
    if (s1 > s0 && s1 == total_len && buf[s1 - 1] == '\n') --s1;  // final newline ends the last line
    line.assign(buf + s0, buf + s1);  // without the newline; NUL-terminated copy for strtod
    bool blank = true;
    for (char c : line)
      if (!std::isspace(static_cast<unsigned char>(c))) {
        blank = false;
        break;
      }
    if (blank) continue;
    const char* p = line.c_str();
    char* end = nullptr;
    auto fail_line = [&](const char* what) {
      out.err_line = li + 1;
      out.err = what;
    };
    const double label = std::strtod(p, &end);
    if (end == p) {
      fail_line("expected numeric label");
      return;
    }
    p = end;
    int64_t cnt = 0, last = -1;
    for (;;) {
      while (*p == ' ' || *p == '\t' || *p == '\r') ++p;
      if (*p == '\0') break;
      const long index = std::strtol(p, &end, 10);
      if (end == p || *end != ':') {
        fail_line("expected <index>:<value>");
        return;
      }
      if (index < 1) {
        fail_line("feature indices are 1-based");
        return;
      }
      p = end + 1;
      const double value = std::strtod(p, &end);
      if (end == p) {
        fail_line("expected numeric feature value");
        return;
      }
      p = end;
      const int32_t zb = static_cast<int32_t>(index - 1);
      if (cnt > 0 && zb <= last) {
        fail_line("feature indices must be strictly increasing");
        return;
      }
      out.col.push_back(zb);
      out.val.push_back(value);
      last = zb;
      ++cnt;
    }
    if (last > out.max_col) out.max_col = last;
    out.row_nnz.push_back(cnt);
    out.y.push_back(label);
  }
}
}  // namespace

int pkrrgpu_load_libsvm(const char* path, int threads, pkrrgpu_dataset** out) {
  try {
    if (!path || !out) fail(PKRRGPU_INVALID, "load_libsvm: null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(PKRRGPU_IO, std::string("cannot open ") + path);
    std::vector<char> buf;
    {
      std::fseek(f, 0, SEEK_END);
      const long len = std::ftell(f);
      std::fseek(f, 0, SEEK_SET);
      buf.resize(static_cast<size_t>(len > 0 ? len : 0));
      const size_t got = len > 0 ? std::fread(buf.data(), 1, buf.size(), f) : 0;
      std::fclose(f);
      buf.resize(got);
    }
    // line starts (std::getline semantics: a trailing newline does not open a line)
    std::vector<int64_t> starts;
    const int64_t L = static_cast<int64_t>(buf.size());
    if (L > 0) starts.push_back(0);
    for (int64_t i = 0; i < L; ++i)
      if (buf[i] == '\n' && i + 1 < L) starts.push_back(i + 1);
    const int64_t nl = static_cast<int64_t>(starts.size());
    int T = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
    if (T < 1) T = 1;
    if (nl < 4096) T = 1;
    std::vector<LibsvmChunk> parts(T);
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
      const int64_t b = nl * t / T, e = nl * (t + 1) / T;
      pool.emplace_back([&, b, e, t] { parse_libsvm_lines(buf.data(), starts, b, e, L, parts[t]); });
    }
    for (auto& th : pool) th.join();
    // the sequential parser stops at the first failing line
    for (const LibsvmChunk& c : parts)
      if (c.err_line >= 0)
        fail(PKRRGPU_IO, std::string(path) + ": parse error at line " + std::to_string(c.err_line) + ": " + c.err);
    auto ds = std::make_unique<pkrrgpu_dataset>();
    int64_t max_col = -1;
    for (const LibsvmChunk& c : parts) {
      for (int64_t k : c.row_nnz) ds->row_ptr.push_back(ds->row_ptr.back() + k);
      ds->col.insert(ds->col.end(), c.col.begin(), c.col.end());
      ds->val.insert(ds->val.end(), c.val.begin(), c.val.end());
      ds->y.insert(ds->y.end(), c.y.begin(), c.y.end());
      max_col = std::max(max_col, c.max_col);
    }
    ds->n = static_cast<int64_t>(ds->y.size());
    ds->d = max_col + 1;
    if (ds->n == 0) fail(PKRRGPU_IO, std::string(path) + ": empty dataset");
    *out = ds.release();
    return PKRRGPU_OK;
  } catch (const Fail& f) {
    return f.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PKRRGPU_IO;
  }
}

int pkrrgpu_dataset_shape(const pkrrgpu_dataset* ds, int64_t* n, int64_t* d, int64_t* nnz) {
  if (!ds) return PKRRGPU_INVALID;
  if (n) *n = ds->n;
  if (d) *d = ds->d;
  if (nnz) *nnz = static_cast<int64_t>(ds->col.size());
  return PKRRGPU_OK;
}

int pkrrgpu_dataset_csr(const pkrrgpu_dataset* ds, int64_t* row_ptr, int32_t* col, double* val, double* y) {
  if (!ds) return PKRRGPU_INVALID;
  if (row_ptr) std::memcpy(row_ptr, ds->row_ptr.data(), sizeof(int64_t) * ds->row_ptr.size());
  if (col) std::memcpy(col, ds->col.data(), sizeof(int32_t) * ds->col.size());
  if (val) std::memcpy(val, ds->val.data(), sizeof(double) * ds->val.size());
  if (y) std::memcpy(y, ds->y.data(), sizeof(double) * ds->y.size());
  return PKRRGPU_OK;
}

int pkrrgpu_dataset_dense(pkrrgpu_ctx* ctx, pkrrgpu_dataset* ds, double* X, double* y) {
  API_BEGIN
  if (!ds || !X) fail(PKRRGPU_INVALID, "dataset_dense: null argument");
  const int64_t n = ds->n, d = ds->d;
  if (!ds->pinned) {
    ck(cudaMallocHost(&ds->pinned, sizeof(double) * static_cast<size_t>(n * d > 0 ? n * d : 1)), "pinned");
    // scatter the CSR rows into dense pinned rows, rows split across host threads
    int T = static_cast<int>(std::thread::hardware_concurrency());
    if (T < 1 || n < 4096) T = 1;
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t)
      pool.emplace_back([ds, n, d, t, T] {
        for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) {
          double* row = ds->pinned + i * d;
          std::fill(row, row + d, 0.0);
          for (int64_t k = ds->row_ptr[i]; k < ds->row_ptr[i + 1]; ++k) row[ds->col[k]] = ds->val[k];
        }
      });
    for (auto& th : pool) th.join();
  }
  cudaStream_t s = ctx->main;
  ck(cudaMemcpyAsync(X, ds->pinned, sizeof(double) * n * d, cudaMemcpyDefault, s), "dense copy");
  if (y) ck(cudaMemcpyAsync(y, ds->y.data(), sizeof(double) * n, cudaMemcpyDefault, s), "label copy");
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

void pkrrgpu_dataset_free(pkrrgpu_dataset* ds) { delete ds; }

// ---- kernel -----------------------------------------------------------------
int pkrrgpu_gram(pkrrgpu_ctx* ctx, const double* A, int64_t na, const double* B, int64_t nb,
                 int64_t d, double sigma, double* K) {
  API_BEGIN
  if (!(sigma > 0.0)) fail(PKRRGPU_INVALID, "gaussian kernel needs sigma > 0");
  if (na <= 0 || nb <= 0 || d <= 0) fail(PKRRGPU_INVALID, "gram: empty input");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const bool same = A == B && na == nb;
  const double* dA = sc.in(A, na * d, s);
  const double* dB = same ? dA : sc.in(B, nb * d, s);
  PartBuf pb;
  part_alloc(sc, pb, nb, d, true, s);
  int64_t* idx = sc.alloc<int64_t>(nb);
  iota_kernel<<<blocks_for(nb), 256, 0, s>>>(idx, nb);
  ctx->counter.launched();
  pk::launch_gather_rows(dB, d, idx, nb, pb.Xp, pb.mp, pb.dp, s, ctx->counter);
  pk::launch_row_norms(pb.Xp, pb.mp, pb.dp, pb.dp, pb.norms, s, ctx->counter);
  if (same) {
    pk::launch_gram_sym(pb.tmX, pb.norms, pb.mp, pb.dp, nb, sigma, pb.K, pb.mp, nullptr, s, ctx->counter);
    ck(cudaMemcpy2DAsync(K, sizeof(double) * nb, pb.K, sizeof(double) * pb.mp, sizeof(double) * nb, na,
                         cudaMemcpyDefault, s),
       "copy K");
  } else {
    QueryBuf qb;
    query_alloc(sc, qb, na, pb.dp, pb.mp, true);
    int64_t* qidx = sc.alloc<int64_t>(na);
    iota_kernel<<<blocks_for(na), 256, 0, s>>>(qidx, na);
    ctx->counter.launched();
    pk::launch_gather_rows(dA, d, qidx, na, qb.Xq, qb.qp, pb.dp, s, ctx->counter);
    pk::launch_row_norms(qb.Xq, qb.qp, pb.dp, pb.dp, qb.norms, s, ctx->counter);
    pk::launch_gram_cross(qb.tmQ, pb.tmX, qb.norms, pb.norms, qb.qp, na, pb.mp, nb, pb.dp, sigma,
                          qb.cross, s, ctx->counter);
    ck(cudaMemcpy2DAsync(K, sizeof(double) * nb, qb.cross, sizeof(double) * pb.mp, sizeof(double) * nb,
                         na, cudaMemcpyDefault, s),
       "copy K");
  }
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

int pkrrgpu_assemble(pkrrgpu_ctx* ctx, const double* K, int64_t m, double lambda, int64_t mult,
                     double* A) {
  API_BEGIN
  if (!(lambda > 0.0)) fail(PKRRGPU_INVALID, "assemble_system: lambda must be > 0");
  if (m <= 0) fail(PKRRGPU_INVALID, "assemble_system: empty matrix");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  // pad to an even count of doubles for the vectorised kernel
  const int64_t mp = round_up(m, 2);
  double* Kp = sc.zeros<double>(mp * mp, s);
  double* Ap = sc.alloc<double>(mp * mp);
  ck(cudaMemcpy2DAsync(Kp, sizeof(double) * mp, K, sizeof(double) * m, sizeof(double) * m, m,
                       cudaMemcpyDefault, s),
     "copy");
  pk::launch_assemble(Kp, Ap, mp, lambda * static_cast<double>(mult), nullptr, s, ctx->counter);
  ck(cudaMemcpy2DAsync(A, sizeof(double) * m, Ap, sizeof(double) * mp, sizeof(double) * m, m,
                       cudaMemcpyDefault, s),
     "copy");
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

// ---- solver -------------------------------------------------------------------
int pkrrgpu_cholesky(pkrrgpu_ctx* ctx, const double* A, int64_t m, double* L, int64_t* npd_pivot) {
  API_BEGIN
  if (m <= 0) fail(PKRRGPU_INVALID, "cholesky: empty matrix");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  PartBuf pb;
  part_alloc(sc, pb, m, 1, false, s);
  ck(cudaMemsetAsync(pb.A, 0, sizeof(double) * pb.mp * pb.mp, s), "memset");
  ck(cudaMemcpy2DAsync(pb.A, sizeof(double) * pb.mp, A, sizeof(double) * m, sizeof(double) * m, m,
                       cudaMemcpyDefault, s),
     "copy A");
  if (pb.mp > m) {
    set_diag_kernel<<<blocks_for(pb.mp - m), 256, 0, s>>>(pb.A, m, pb.mp, 1.0);
    ctx->counter.launched();
  }
  int* status = sc.zeros<int>(2, s);
  pk::launch_potrf(pb.A, pb.tmA, pb.tmLinv, pb.Linv, pb.mp, m, status, s, ctx->counter, pb.slices, pb.exps,
                   ctx->aux_main, true);
  std::vector<int> st = to_host(status, 2, s);
  if (st[0]) {
    if (npd_pivot) *npd_pivot = st[1];
    fail(PKRRGPU_NPD, "matrix not positive definite: pivot " + std::to_string(st[1]));
  }
  pk::launch_zero_upper(pb.A, pb.mp, s, ctx->counter);
  ck(cudaMemcpy2DAsync(L, sizeof(double) * m, pb.A, sizeof(double) * pb.mp, sizeof(double) * m, m,
                       cudaMemcpyDefault, s),
     "copy L");
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

int pkrrgpu_solve_spd(pkrrgpu_ctx* ctx, const double* L, int64_t m, const double* b, double* x) {
  API_BEGIN
  if (m <= 0) fail(PKRRGPU_INVALID, "solve_spd: size mismatch");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  PartBuf pb;
  part_alloc(sc, pb, m, 1, false, s);
  ck(cudaMemsetAsync(pb.A, 0, sizeof(double) * pb.mp * pb.mp, s), "memset");
  ck(cudaMemcpy2DAsync(pb.A, sizeof(double) * pb.mp, L, sizeof(double) * m, sizeof(double) * m, m,
                       cudaMemcpyDefault, s),
     "copy L");
  if (pb.mp > m) {
    set_diag_kernel<<<blocks_for(pb.mp - m), 256, 0, s>>>(pb.A, m, pb.mp, 1.0);
    ctx->counter.launched();
  }
  ck(cudaMemsetAsync(pb.yp, 0, sizeof(double) * pb.mp, s), "memset");
  ck(cudaMemcpyAsync(pb.yp, b, sizeof(double) * m, cudaMemcpyDefault, s), "copy b");
  pk::launch_diag_inverses(pb.A, pb.mp, pb.Linv, s, ctx->counter);
  pk::launch_trsv(pb.A, pb.Linv, pb.mp, pb.yp, pb.z, pb.alpha, pb.scratch, nullptr, s, ctx->counter);
  copy_out(x, pb.alpha, m, s);
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

int pkrrgpu_train_krr(pkrrgpu_ctx* ctx, const double* X, const double* y, int64_t m, int64_t d,
                      double sigma, double lambda, double* alpha, double* residual,
                      int64_t* npd_pivot) {
  API_BEGIN
  if (m <= 0) fail(PKRRGPU_INVALID, "train_krr: empty dataset");
  if (!(lambda > 0.0)) fail(PKRRGPU_INVALID, "train_krr: lambda must be > 0");
  if (!(sigma > 0.0)) fail(PKRRGPU_INVALID, "gaussian kernel needs sigma > 0");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dX = sc.in(X, m * d, s);
  const double* dy = sc.in(y, m, s);
  PartBuf pb;
  part_alloc(sc, pb, m, d, true, s);
  int64_t* idx = sc.alloc<int64_t>(m);
  iota_kernel<<<blocks_for(m), 256, 0, s>>>(idx, m);
  ctx->counter.launched();
  part_load(ctx, pb, dX, dy, d, idx, s);
  const bool assembled = pk::launch_gram_sym(pb.tmX, pb.norms, pb.mp, pb.dp, m, sigma, pb.K, pb.mp, nullptr, s,
                                             ctx->counter, false, pb.A, lambda * static_cast<double>(m));
  int* status = sc.zeros<int>(2, s);
  double* res = sc.zeros<double>(2, s);
  part_solve(ctx, pb, lambda, status, res, s, ctx->aux_main, true, assembled);
  std::vector<int> st = to_host(status, 2, s);
  if (st[0]) {
    if (npd_pivot) *npd_pivot = st[1];
    fail(PKRRGPU_NPD, "matrix not positive definite: pivot " + std::to_string(st[1]));
  }
  copy_out(alpha, pb.alpha, m, s);
  if (residual) *residual = to_host(res, 2, s)[1];  // solver.cpp:119 form
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

int pkrrgpu_predict(pkrrgpu_ctx* ctx, const double* S, const double* alpha, int64_t m, int64_t d,
                    double sigma, const double* Q, int64_t q, double* out) {
  API_BEGIN
  if (m <= 0 || q <= 0) fail(PKRRGPU_INVALID, "predict: empty input");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dS = sc.in(S, m * d, s);
  const double* dQ = sc.in(Q, q * d, s);
  PartBuf pb;
  pb.m = m;
  pb.mp = round_up(m, kNB);
  pb.dp = round_up(d, 16);
  pb.Xp = sc.alloc<double>(pb.mp * pb.dp);
  pb.norms = sc.alloc<double>(pb.mp);
  pb.alpha = sc.zeros<double>(pb.mp, s);
  if (!pk::make_tmap(&pb.tmX, pb.Xp, pb.mp, pb.dp, pb.dp)) fail(PKRRGPU_CUDA, "tensor map");
  ck(cudaMemcpyAsync(pb.alpha, alpha, sizeof(double) * m, cudaMemcpyDefault, s), "copy alpha");
  int64_t* idx = sc.alloc<int64_t>(std::max(m, q));
  iota_kernel<<<blocks_for(std::max(m, q)), 256, 0, s>>>(idx, std::max(m, q));
  ctx->counter.launched();
  pk::launch_gather_rows(dS, d, idx, m, pb.Xp, pb.mp, pb.dp, s, ctx->counter);
  pk::launch_row_norms(pb.Xp, pb.mp, pb.dp, pb.dp, pb.norms, s, ctx->counter);
  QueryBuf qb;
  query_alloc(sc, qb, q, pb.dp, pb.mp);
  pk::launch_gather_rows(dQ, d, idx, q, qb.Xq, qb.qp, pb.dp, s, ctx->counter);
  pk::launch_row_norms(qb.Xq, qb.qp, pb.dp, pb.dp, qb.norms, s, ctx->counter);
  pk::launch_predict_fused(qb.tmQ, pb.tmX, qb.norms, pb.norms, qb.qp, q, pb.mp, m, pb.dp, sigma, pb.alpha,
                           qb.partial, qb.pred, nullptr, s, ctx->counter);
  copy_out(out, qb.pred, q, s);
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

// ---- clustering -------------------------------------------------------------
int pkrrgpu_kmeans(pkrrgpu_ctx* ctx, const double* X, int64_t n, int64_t d, int k, uint64_t seed,
                   double threshold, int max_iters, int32_t* membership, double* centers,
                   int64_t* sizes, int* iterations) {
  API_BEGIN
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dX = sc.in(X, n * d, s);
  double* xnorm = sc.alloc<double>(n);
  pk::launch_row_norms(dX, n, d, d, xnorm, s, ctx->counter);
  ClusterOut co;
  kmeans_device(ctx, sc, dX, n, d, k, seed, threshold, max_iters, xnorm, co);
  copy_out(membership, co.label, n, s);
  copy_out(centers, co.centers, static_cast<int64_t>(k) * d, s);
  if (sizes) std::memcpy(sizes, co.h_sizes.data(), sizeof(int64_t) * k);
  if (iterations) *iterations = co.iterations;
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

int pkrrgpu_kbalance(pkrrgpu_ctx* ctx, const double* X, int64_t n, int64_t d, int k, uint64_t seed,
                     double threshold, int max_iters, int recompute, int32_t* membership,
                     double* centers, int64_t* sizes) {
  API_BEGIN
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dX = sc.in(X, n * d, s);
  double* xnorm = sc.alloc<double>(n);
  pk::launch_row_norms(dX, n, d, d, xnorm, s, ctx->counter);
  ClusterOut co;
  kbalance_device(ctx, sc, dX, n, d, k, seed, threshold, max_iters, recompute != 0, xnorm, co);
  copy_out(membership, co.label, n, s);
  copy_out(centers, co.centers, static_cast<int64_t>(k) * d, s);
  if (sizes) std::memcpy(sizes, co.h_sizes.data(), sizeof(int64_t) * k);
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

int pkrrgpu_nearest_center(pkrrgpu_ctx* ctx, const double* centers, int k, int64_t d,
                           const double* Q, int64_t q, int32_t* out) {
  API_BEGIN
  if (k < 1) fail(PKRRGPU_INVALID, "nearest_center: no centers");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dC = sc.in(centers, static_cast<int64_t>(k) * d, s);
  const double* dQ = sc.in(Q, q * d, s);
  RouteOut ro;
  route_rows(ctx, sc, dQ, q, d, dC, k, ro);
  copy_out(out, ro.route, q, s);
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

// ---- strategies ---------------------------------------------------------------
int pkrrgpu_make_partition(pkrrgpu_ctx* ctx, int strategy, const double* X, int64_t n, int64_t d,
                           int64_t p, uint64_t seed, int32_t* part_of, int64_t* order,
                           double* centers, int64_t* p_out) {
  API_BEGIN
  if (strategy < 0 || strategy > 7) fail(PKRRGPU_INVALID, "unknown strategy");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dX = sc.in(X, n * d, s);
  PartitionOut po;
  make_partition_device(ctx, sc, strategy, dX, n, d, p, seed, 0.01, 100, po);
  copy_out(part_of, po.part_of, n, s);
  copy_out(order, po.order, n, s);
  if (centers && po.centers) copy_out(centers, po.centers, po.p * d, s);
  if (p_out) *p_out = po.p;
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

}  // extern "C"

// ---- trained models (TrainedPartitions) ---------------------------------------
struct pkrrgpu_models {
  pkrrgpu_ctx* ctx = nullptr;
  int64_t p = 0, d = 0, dp = 0;
  double sigma = 1.0;
  std::vector<int64_t> m, mp;
  std::vector<double*> Xp, norms, alpha;
  std::vector<CUtensorMap> tmX;
  std::vector<double> residual;
  double* centers = nullptr;  // p x d (null for whole/random partitions)
  int predictor = 2;
};

extern "C" {

}  // extern "C"

namespace {

// train_partitions core (strategies.cpp:104-133): every part of `po` trained
// concurrently, largest first on the highest-priority streams (LPT over the context's
// 8 part streams, each with its lookahead companion); the support rows, norms and
// alpha are kept resident as the models (KrrModel, solver.hpp:37-49).
pkrrgpu_models* train_models(pkrrgpu_ctx* ctx, Scope& sc, const double* dX, const double* dy, int64_t d,
                             const PartitionOut& po, double sigma, double lambda, int predictor,
                             int64_t* failed_part, int64_t* npd_pivot) {
  cudaStream_t s = ctx->main;
  for (int64_t t = 0; t < po.p; ++t)
    if (po.sizes[t] == 0) fail(PKRRGPU_INVALID, "train_partitions: empty part");
  std::vector<PartBuf> parts(po.p);
  int* status = sc.zeros<int>(2 * po.p, s);
  double* res = sc.zeros<double>(2 * po.p, s);
  cudaEvent_t ready;
  ck(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
  ck(cudaEventRecord(ready, s), "event");
  std::vector<int64_t> by_size(po.p);
  for (int64_t t = 0; t < po.p; ++t) by_size[t] = t;
  std::stable_sort(by_size.begin(), by_size.end(), [&](int64_t x, int64_t y) { return po.sizes[x] > po.sizes[y]; });
  const size_t S = ctx->work.size();
  for (size_t i = 0; i < by_size.size(); ++i) {
    const int64_t t = by_size[i];
    cudaStream_t ws = ctx->work[i % S];
    ck(cudaStreamWaitEvent(ws, ready, 0), "wait");
    PartBuf& pb = parts[t];
    part_alloc(sc, pb, po.sizes[t], d, true, ws);
    part_load(ctx, pb, dX, dy, d, po.order + po.start[t], ws);
    const bool assembled = pk::launch_gram_sym(pb.tmX, pb.norms, pb.mp, pb.dp, pb.m, sigma, pb.K, pb.mp, nullptr, ws,
                                               ctx->counter, false, pb.A, lambda * static_cast<double>(pb.m));
    part_solve(ctx, pb, lambda, status + 2 * t, res + 2 * t, ws, ctx->aux[i % S], po.p == 1, assembled);
  }
  ck(cudaEventDestroy(ready), "event");
  ck(cudaDeviceSynchronize(), "train");
  std::vector<int> st = to_host(status, 2 * po.p, s);
  std::vector<double> rh = to_host(res, 2 * po.p, s);
  for (int64_t t = 0; t < po.p; ++t)
    if (st[2 * t]) {
      if (failed_part) *failed_part = t;
      if (npd_pivot) *npd_pivot = st[2 * t + 1];
      fail(PKRRGPU_NPD, "partition " + std::to_string(t) + ": matrix not positive definite: pivot " +
                            std::to_string(st[2 * t + 1]));
    }
  auto mod = std::make_unique<pkrrgpu_models>();
  mod->ctx = ctx;
  mod->p = po.p;
  mod->d = d;
  mod->dp = round_up(d, 16);
  mod->sigma = sigma;
  mod->predictor = predictor;
  for (int64_t t = 0; t < po.p; ++t) {
    PartBuf& pb = parts[t];
    mod->m.push_back(pb.m);
    mod->mp.push_back(pb.mp);
    double* x = static_cast<double*>(ctx->alloc(sizeof(double) * pb.mp * pb.dp));
    double* nm = static_cast<double*>(ctx->alloc(sizeof(double) * pb.mp));
    double* al = static_cast<double*>(ctx->alloc(sizeof(double) * pb.mp));
    mod->Xp.push_back(x);
    mod->norms.push_back(nm);
    mod->alpha.push_back(al);
    ck(cudaMemcpyAsync(x, pb.Xp, sizeof(double) * pb.mp * pb.dp, cudaMemcpyDeviceToDevice, s), "copy");
    ck(cudaMemcpyAsync(nm, pb.norms, sizeof(double) * pb.mp, cudaMemcpyDeviceToDevice, s), "copy");
    ck(cudaMemcpyAsync(al, pb.alpha, sizeof(double) * pb.mp, cudaMemcpyDeviceToDevice, s), "copy");
    CUtensorMap tm;
    if (!pk::make_tmap(&tm, x, pb.mp, pb.dp, pb.dp)) fail(PKRRGPU_CUDA, "tensor map");
    mod->tmX.push_back(tm);
    mod->residual.push_back(rh[2 * t + 1]);
  }
  if (po.centers) {
    mod->centers = static_cast<double*>(ctx->alloc(sizeof(double) * po.p * d));
    ck(cudaMemcpyAsync(mod->centers, po.centers, sizeof(double) * po.p * d, cudaMemcpyDeviceToDevice, s), "copy");
  }
  ck(cudaStreamSynchronize(s), "sync");
  return mod.release();
}

// the caller's PartitionSet (strategies.hpp:31-36) as a device PartitionOut: part t =
// rows[start_t .. start_t + sizes[t]) in the caller's order (make_partition keeps train
// row order, strategies.cpp:97-99; a random partition keeps its permutation order)
void partition_from_lists(pkrrgpu_ctx* ctx, Scope& sc, const int64_t* rows, const int64_t* sizes, int64_t p,
                          int64_t n, const double* centers, int64_t d, PartitionOut& po) {
  cudaStream_t s = ctx->main;
  if (p < 1) fail(PKRRGPU_INVALID, "partition: need p >= 1");
  po.p = p;
  po.sizes.assign(sizes, sizes + p);
  po.start.assign(p, 0);
  int64_t total = 0;
  for (int64_t t = 0; t < p; ++t) {
    if (sizes[t] <= 0) fail(PKRRGPU_INVALID, "train_partitions: empty part");
    po.start[t] = total;
    total += sizes[t];
  }
  std::vector<int64_t> h(total);
  ck(cudaMemcpy(h.data(), rows, sizeof(int64_t) * total, cudaMemcpyDefault), "copy rows");
  for (int64_t i = 0; i < total; ++i)
    if (h[i] < 0 || h[i] >= n) fail(PKRRGPU_INVALID, "train_partitions: row index out of range");
  po.order = sc.upload(h, s);
  po.centers = centers ? const_cast<double*>(sc.in(centers, p * d, s)) : nullptr;
}

}  // namespace

extern "C" {

int pkrrgpu_train_partitions(pkrrgpu_ctx* ctx, int strategy, const double* X, const double* y,
                             int64_t n, int64_t d, int64_t p, uint64_t seed, double sigma,
                             double lambda, pkrrgpu_models** out, int64_t* failed_part,
                             int64_t* npd_pivot) {
  API_BEGIN
  if (!out) fail(PKRRGPU_INVALID, "null out");
  if (!(lambda > 0.0)) fail(PKRRGPU_INVALID, "train_krr: lambda must be > 0");
  if (!(sigma > 0.0)) fail(PKRRGPU_INVALID, "gaussian kernel needs sigma > 0");
  if (strategy < 0 || strategy > 7) fail(PKRRGPU_INVALID, "unknown strategy");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dX = sc.in(X, n * d, s);
  const double* dy = sc.in(y, n, s);
  PartitionOut po;
  make_partition_device(ctx, sc, strategy, dX, n, d, p, seed, 0.01, 100, po);
  *out = train_models(ctx, sc, dX, dy, d, po, sigma, lambda, predictor_of(strategy), failed_part, npd_pivot);
  API_END
}

int pkrrgpu_train_parts(pkrrgpu_ctx* ctx, const double* X, const double* y, int64_t n, int64_t d,
                        const int64_t* rows, const int64_t* sizes, int64_t p, const double* centers, double sigma,
                        double lambda, pkrrgpu_models** out, int64_t* failed_part, int64_t* npd_pivot) {
  API_BEGIN
  if (!out || !rows || !sizes) fail(PKRRGPU_INVALID, "null argument");
  if (n <= 0 || d <= 0) fail(PKRRGPU_INVALID, "train_partitions: empty dataset");
  if (!(lambda > 0.0)) fail(PKRRGPU_INVALID, "train_krr: lambda must be > 0");
  if (!(sigma > 0.0)) fail(PKRRGPU_INVALID, "gaussian kernel needs sigma > 0");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dX = sc.in(X, n * d, s);
  const double* dy = sc.in(y, n, s);
  PartitionOut po;
  partition_from_lists(ctx, sc, rows, sizes, p, n, centers, d, po);
  *out = train_models(ctx, sc, dX, dy, d, po, sigma, lambda, centers ? 2 : 0, failed_part, npd_pivot);
  API_END
}

int pkrrgpu_models_import(pkrrgpu_ctx* ctx, int64_t p, int64_t d, const int64_t* sizes, const double* S,
                          const double* alpha, const double* centers, double sigma, pkrrgpu_models** out) {
  API_BEGIN
  if (!out || !sizes || !S || !alpha || p < 1 || d <= 0) fail(PKRRGPU_INVALID, "models_import: bad arguments");
  if (!(sigma > 0.0)) fail(PKRRGPU_INVALID, "gaussian kernel needs sigma > 0");
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  int64_t total = 0;
  for (int64_t t = 0; t < p; ++t) {
    if (sizes[t] <= 0) fail(PKRRGPU_INVALID, "models_import: empty model");
    total += sizes[t];
  }
  const double* dS = sc.in(S, total * d, s);
  const double* dA = sc.in(alpha, total, s);
  auto mod = std::make_unique<pkrrgpu_models>();
  mod->ctx = ctx;
  mod->p = p;
  mod->d = d;
  mod->dp = round_up(d, 16);
  mod->sigma = sigma;
  mod->predictor = centers ? 2 : 0;
  int64_t at = 0;
  for (int64_t t = 0; t < p; ++t) {
    const int64_t m = sizes[t], mp = round_up(m, kNB);
    double* x = static_cast<double*>(ctx->alloc(sizeof(double) * mp * mod->dp));
    double* nm = static_cast<double*>(ctx->alloc(sizeof(double) * mp));
    double* al = static_cast<double*>(ctx->alloc(sizeof(double) * mp));
    mod->m.push_back(m);
    mod->mp.push_back(mp);
    mod->Xp.push_back(x);
    mod->norms.push_back(nm);
    mod->alpha.push_back(al);
    int64_t* idx = sc.alloc<int64_t>(m);
    iota_kernel<<<blocks_for(m), 256, 0, s>>>(idx, m);
    ctx->counter.launched();
    pk::launch_gather_rows(dS + at * d, d, idx, m, x, mp, mod->dp, s, ctx->counter);
    pk::launch_row_norms(x, mp, mod->dp, mod->dp, nm, s, ctx->counter);
    ck(cudaMemsetAsync(al, 0, sizeof(double) * mp, s), "memset");
    ck(cudaMemcpyAsync(al, dA + at, sizeof(double) * m, cudaMemcpyDeviceToDevice, s), "copy alpha");
    CUtensorMap tm;
    if (!pk::make_tmap(&tm, x, mp, mod->dp, mod->dp)) fail(PKRRGPU_CUDA, "tensor map");
    mod->tmX.push_back(tm);
    mod->residual.push_back(0.0);
    at += m;
  }
  if (centers) {
    mod->centers = static_cast<double*>(ctx->alloc(sizeof(double) * p * d));
    ck(cudaMemcpyAsync(mod->centers, centers, sizeof(double) * p * d, cudaMemcpyDefault, s), "copy centers");
  }
  ck(cudaStreamSynchronize(s), "sync");
  *out = mod.release();
  API_END
}

int64_t pkrrgpu_models_count(const pkrrgpu_models* m) { return m ? m->p : 0; }
int64_t pkrrgpu_models_size(const pkrrgpu_models* m, int64_t t) {
  return (m && t >= 0 && t < m->p) ? m->m[t] : -1;
}
int pkrrgpu_models_alpha(const pkrrgpu_models* m, int64_t t, double* alpha) {
  if (!m || t < 0 || t >= m->p || !alpha) return PKRRGPU_INVALID;
  cudaSetDevice(m->ctx->device);
  return cudaMemcpy(alpha, m->alpha[t], sizeof(double) * m->m[t], cudaMemcpyDefault) == cudaSuccess
             ? PKRRGPU_OK
             : PKRRGPU_CUDA;
}
int pkrrgpu_models_residual(const pkrrgpu_models* m, int64_t t, double* r) {
  if (!m || t < 0 || t >= m->p || !r) return PKRRGPU_INVALID;
  *r = m->residual[t];
  return PKRRGPU_OK;
}
void pkrrgpu_models_free(pkrrgpu_models* m) {
  if (!m) return;
  cudaSetDevice(m->ctx->device);
  cudaDeviceSynchronize();
  for (auto* p : m->Xp) m->ctx->release(p);
  for (auto* p : m->norms) m->ctx->release(p);
  for (auto* p : m->alpha) m->ctx->release(p);
  if (m->centers) m->ctx->release(m->centers);
  delete m;
}

int pkrrgpu_predict_nearest(pkrrgpu_ctx* ctx, const pkrrgpu_models* models, const double* Q,
                            int64_t q, double* out) {
  API_BEGIN
  if (!models || models->p < 1) fail(PKRRGPU_INVALID, "predict_nearest: no models");
  if (!models->centers)
    fail(PKRRGPU_INVALID, "predict_nearest: centers undefined for this partitioning");
  if (models->ctx->device != ctx->device) fail(PKRRGPU_INVALID, "predict_nearest: models live on another device");
  if (q <= 0) API_RETURN_OK;
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const int64_t d = models->d, dp = models->dp;
  const double* dQ = sc.in(Q, q * d, s);
  RouteOut ro;
  route_rows(ctx, sc, dQ, q, d, models->centers, static_cast<int>(models->p), ro);
  double* pred_all = sc.alloc<double>(q);
  double* ydummy = sc.zeros<double>(q, s);
  double* sse = sc.alloc<double>(models->p);
  cudaEvent_t ready;
  ck(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
  ck(cudaEventRecord(ready, s), "event");
  for (int64_t t = 0; t < models->p; ++t) {
    const int64_t cnt = ro.sizes[t];
    if (cnt == 0) continue;
    cudaStream_t ws = ctx->work[t % ctx->work.size()];
    ck(cudaStreamWaitEvent(ws, ready, 0), "wait");
    QueryBuf qb;
    query_alloc(sc, qb, cnt, dp, models->mp[t]);
    const int64_t* rows = ro.members + ro.start[t];
    pk::launch_gather_rows(dQ, d, rows, cnt, qb.Xq, qb.qp, dp, ws, ctx->counter);
    pk::launch_row_norms(qb.Xq, qb.qp, dp, dp, qb.norms, ws, ctx->counter);
    pk::launch_predict_fused(qb.tmQ, models->tmX[t], qb.norms, models->norms[t], qb.qp, cnt, models->mp[t],
                             models->m[t], dp, models->sigma, models->alpha[t], qb.partial, qb.pred, nullptr, ws,
                             ctx->counter);
    pk::launch_sse_scatter(qb.pred, rows, cnt, ydummy, pred_all, sse + t, nullptr, ws, ctx->counter);
  }
  ck(cudaEventDestroy(ready), "event");
  ck(cudaDeviceSynchronize(), "predict");
  copy_out(out, pred_all, q, s);
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

int pkrrgpu_models_predict(pkrrgpu_ctx* ctx, const pkrrgpu_models* models, int64_t part, const double* Q,
                           int64_t q, double* out) {
  API_BEGIN
  if (!models || models->p < 1) fail(PKRRGPU_INVALID, "predict: no models");
  if (part < -1 || part >= models->p) fail(PKRRGPU_INVALID, "predict: no such model");
  if (models->ctx->device != ctx->device) fail(PKRRGPU_INVALID, "predict: models live on another device");
  if (q <= 0) API_RETURN_OK;
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const int64_t d = models->d, dp = models->dp;
  const double* dQ = sc.in(Q, q * d, s);
  const int64_t t0 = part < 0 ? 0 : part, t1 = part < 0 ? models->p : part + 1;
  double* dout = sc.alloc<double>((t1 - t0) * q);
  int64_t* idx = sc.alloc<int64_t>(q);
  iota_kernel<<<blocks_for(q), 256, 0, s>>>(idx, q);
  ctx->counter.launched();
  QueryBuf qb0;
  query_alloc(sc, qb0, q, dp, kNB);
  pk::launch_gather_rows(dQ, d, idx, q, qb0.Xq, qb0.qp, dp, s, ctx->counter);
  pk::launch_row_norms(qb0.Xq, qb0.qp, dp, dp, qb0.norms, s, ctx->counter);
  cudaEvent_t ready;
  ck(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
  ck(cudaEventRecord(ready, s), "event");
  for (int64_t t = t0; t < t1; ++t) {
    cudaStream_t ws = ctx->work[(t - t0) % ctx->work.size()];
    ck(cudaStreamWaitEvent(ws, ready, 0), "wait");
    double* partial = sc.alloc<double>(pk::predict_partial_elems(qb0.qp, models->mp[t]));
    pk::launch_predict_fused(qb0.tmQ, models->tmX[t], qb0.norms, models->norms[t], qb0.qp, q, models->mp[t],
                             models->m[t], dp, models->sigma, models->alpha[t], partial, dout + (t - t0) * q,
                             nullptr, ws, ctx->counter);
  }
  ck(cudaEventDestroy(ready), "event");
  ck(cudaDeviceSynchronize(), "predict");
  copy_out(out, dout, (t1 - t0) * q, s);
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

int pkrrgpu_models_centers(const pkrrgpu_models* m, double* centers) {
  if (!m || !centers) return PKRRGPU_INVALID;
  if (!m->centers) return PKRRGPU_INVALID;
  cudaSetDevice(m->ctx->device);
  return cudaMemcpy(centers, m->centers, sizeof(double) * m->p * m->d, cudaMemcpyDefault) == cudaSuccess
             ? PKRRGPU_OK
             : PKRRGPU_CUDA;
}

int pkrrgpu_combine(pkrrgpu_ctx* ctx, int strategy, int64_t p, int64_t t, int64_t ncell, const double* pred,
                    const double* y, const uint8_t* cell_failed, double* cell_mse, int64_t* best_index,
                    double* best_pred) {
  API_BEGIN
  if (strategy < 0 || strategy > 7) fail(PKRRGPU_INVALID, "unknown strategy");
  if (t <= 0 || ncell <= 0 || p < 1 || !pred || !y) fail(PKRRGPU_INVALID, "combine: bad arguments");
  const int predictor = predictor_of(strategy);
  const int64_t P = predictor == 0 || predictor == 2 ? 1 : p;
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  const double* dp = sc.in(pred, ncell * P * t, s);
  const double* dy = sc.in(y, t, s);
  std::vector<uint8_t> cfail(ncell, 0);
  if (cell_failed) std::memcpy(cfail.data(), cell_failed, ncell);
  std::vector<double> cmse;
  const int64_t b = combine_cells(ctx, sc, predictor, P, t, ncell, dp, dy, cfail, cmse, best_pred);
  if (cell_mse) std::memcpy(cell_mse, cmse.data(), sizeof(double) * ncell);
  if (best_index) *best_index = b;
  ck(cudaStreamSynchronize(s), "sync");
  API_END
}

// ---- grid search (strategies.cpp:343-507) -----------------------------------
int pkrrgpu_grid_search_ex(pkrrgpu_ctx* ctx, const pkrrgpu_grid_args* a, pkrrgpu_grid_out* o) {
  API_BEGIN
  if (!a || !o) fail(PKRRGPU_INVALID, "null args");
  if (a->n_lambdas <= 0 || a->n_sigmas <= 0) fail(PKRRGPU_INVALID, "grid_search: empty grid");
  if (a->n <= 0 || a->t <= 0) fail(PKRRGPU_INVALID, "grid_search: empty dataset");
  if (a->strategy < 0 || a->strategy > 7) fail(PKRRGPU_INVALID, "unknown strategy");
  for (int64_t i = 0; i < a->n_lambdas; ++i)
    if (!(a->lambdas[i] > 0.0)) fail(PKRRGPU_INVALID, "assemble_system: lambda must be > 0");
  for (int64_t i = 0; i < a->n_sigmas; ++i)
    if (!(a->sigmas[i] > 0.0)) fail(PKRRGPU_INVALID, "gaussian kernel needs sigma > 0");
  const int world = a->world > 0 ? a->world : 1, rank = a->rank;
  const int64_t n = a->n, d = a->d, t = a->t, te = (a->X_eval && a->t_eval > 0) ? a->t_eval : 0;
  const int64_t nl = a->n_lambdas, ns = a->n_sigmas, ncell = nl * ns;
  const int predictor = predictor_of(a->strategy);
  Scope sc(ctx);
  cudaStream_t s = ctx->main;
  finalize_timings(ctx);  // the previous call's pooled events are about to be re-recorded
  ctx->ev_next = 0;
  struct {
    cudaEvent_t a, b;
  } t_all{ctx->pool_event(), ctx->pool_event()}, t_part{ctx->pool_event(), ctx->pool_event()};
  ck(cudaEventRecord(t_all.a, s), "event");
  // PKRR_TRACE_HOST=1: host-side timestamps of the grid call's phases (stderr)
  static const bool htrace = std::getenv("PKRR_TRACE_HOST") != nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  auto hmark = [&](const char* what) {
    if (htrace)
      fprintf(stderr, "pkrr host %8.3f ms  %s\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count(), what);
  };

  const double* dX = sc.in(a->X_train, n * d, s);
  const double* dy = sc.in(a->y_train, n, s);
  const double* dXt = sc.in(a->X_test, t * d, s);
  const double* dyt = sc.in(a->y_test, t, s);
  const double* dXe = te ? sc.in(a->X_eval, te * d, s) : nullptr;
  const double* dye = te ? sc.in(a->y_eval, te, s) : nullptr;

  // ---- partition (once; sigma independent) ----
  ck(cudaEventRecord(t_part.a, s), "event");
  PartitionOut po;
  const double thr = a->km_max_iters > 0 ? a->km_threshold : 0.01;
  const int iters = a->km_max_iters > 0 ? a->km_max_iters : 100;
  hmark("inputs enqueued");
  Exchange ex;
  ex.fn = a->allgather;
  ex.user = a->allgather_user;
  ex.rank = rank;
  ex.world = world;
  make_partition_device(ctx, sc, a->strategy, dX, n, d, a->p, a->seed, thr, iters, po, &ex);
  hmark("partition returned");
  const int64_t p = po.p;
  for (int64_t q = 0; q < p; ++q)
    if (po.sizes[q] == 0) fail(PKRRGPU_INVALID, "train_partitions: empty part");
  // ---- targets (strategies.cpp:370-381) ----
  RouteOut rt, re;
  int64_t* iota_t = nullptr;
  int64_t* iota_e = nullptr;
  if (predictor == 2) {
    if (!po.centers) fail(PKRRGPU_INVALID, "grid_search: nearest predictor needs centers");
    route_rows(ctx, sc, dXt, t, d, po.centers, static_cast<int>(p), rt);
    if (te) route_rows(ctx, sc, dXe, te, d, po.centers, static_cast<int>(p), re);
  } else {
    iota_t = sc.alloc<int64_t>(t);
    iota_kernel<<<blocks_for(t), 256, 0, s>>>(iota_t, t);
    ctx->counter.launched();
    if (te) {
      iota_e = sc.alloc<int64_t>(te);
      iota_kernel<<<blocks_for(te), 256, 0, s>>>(iota_e, te);
      ctx->counter.launched();
    }
  }
  ck(cudaEventRecord(t_part.b, s), "event");
  hmark("routing returned");

  // ---- per-part buffers for the parts this rank owns ----
  // Ownership across ranks: LPT on the Cholesky cost m^3 (largest part first to the
  // least-loaded rank, ties to the lower index / rank) -- every rank holds the same
  // partition, so every rank computes the same assignment (sharding.owned_parts).
  std::vector<int64_t> owned;
  {
    std::vector<int64_t> ord(p);
    for (int64_t q = 0; q < p; ++q) ord[q] = q;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return po.sizes[x] > po.sizes[y]; });
    std::vector<double> rload(world, 0.0);
    std::vector<int> owner(p, 0);
    for (int64_t q : ord) {
      int best = 0;
      for (int r = 1; r < world; ++r)
        if (rload[r] < rload[best]) best = r;
      owner[q] = best;
      const double m = static_cast<double>(po.sizes[q]);
      rload[best] += m * m * m;
    }
    for (int64_t q = 0; q < p; ++q)
      if (owner[q] == rank) owned.push_back(q);
  }
  const int64_t dp = round_up(d, 16);
  std::vector<PartBuf> parts(p);
  std::vector<QueryBuf> qt(p), qe(p);
  std::vector<int64_t> tcount(p), ecount(p);
  std::vector<const int64_t*> tpos(p), epos(p);
  for (int64_t q = 0; q < p; ++q) {
    tcount[q] = predictor == 2 ? rt.sizes[q] : t;
    tpos[q] = predictor == 2 ? rt.members + rt.start[q] : iota_t;
    ecount[q] = te ? (predictor == 2 ? re.sizes[q] : te) : 0;
    epos[q] = te ? (predictor == 2 ? re.members + re.start[q] : iota_e) : nullptr;
  }
  // per (cell, part) result slots: [status0, status1] ints; [res_grid, res_train, sse, esse] doubles
  int* dstatus = sc.zeros<int>(ncell * p * 2, s);
  double* dres = sc.zeros<double>(ncell * p * 4, s);
  // per-cell predictions in test order (nearest/whole) or per-part (average/oracle)
  const int64_t pp_parts = predictor == 2 || predictor == 0 ? 1 : p;
  double* pred_t = sc.zeros<double>(ncell * pp_parts * t, s);
  double* pred_e = te ? sc.zeros<double>(ncell * pp_parts * te, s) : nullptr;
  double* comb = world == 1 ? sc.alloc<double>(ncell * t) : nullptr;
  double* dmse = world == 1 ? sc.alloc<double>(ncell) : nullptr;
  double* comb_e = world == 1 && te ? sc.alloc<double>(ncell * te) : nullptr;
  double* dmse_e = world == 1 && te ? sc.alloc<double>(ncell) : nullptr;
  // the part streams' first work (buffer memsets, row gathers from the partition's order
  // array and the uploaded inputs) is ordered after everything enqueued on s so far by
  // this event -- not by a host sync, which left the GPU idle while the host set up parts
  cudaEvent_t e_pre;
  ck(cudaEventCreateWithFlags(&e_pre, cudaEventDisableTiming), "event");
  ck(cudaEventRecord(e_pre, s), "event");
  hmark("result slots ready");

  double f_chol = 0, f_gram = 0, f_other = 0;
  size_t S = ctx->work.size();
  if (const char* e = std::getenv("PKRR_STREAMS")) S = std::max<size_t>(1, std::min<size_t>(S, std::atoi(e)));
  // LPT: parts (largest first) go to the least-loaded stream (load = m^3 per cell).
  // Uneven loads (KKRR2) -> graded stream priorities, the most-loaded stream first,
  // so the critical part wins the block scheduler; balanced loads -> equal priority.
  std::vector<int64_t> by_size(owned);
  std::stable_sort(by_size.begin(), by_size.end(),
                   [&](int64_t x, int64_t y) { return po.sizes[x] > po.sizes[y]; });
  std::vector<size_t> slot(p, 0);
  std::vector<double> load(S, 0.0);
  for (int64_t q : by_size) {
    size_t best = 0;
    for (size_t i = 1; i < S; ++i)
      if (load[i] < load[best]) best = i;
    slot[q] = best;
    load[best] += static_cast<double>(po.sizes[q]) * po.sizes[q] * po.sizes[q];
  }
  std::vector<size_t> order_by_load(S);
  for (size_t i = 0; i < S; ++i) order_by_load[i] = i;
  std::stable_sort(order_by_load.begin(), order_by_load.end(),
                   [&](size_t x, size_t y) { return load[x] > load[y]; });
  std::vector<size_t> rank_of(S);
  for (size_t r = 0; r < S; ++r) rank_of[order_by_load[r]] = r;
  std::vector<double> nz;
  for (double l : load)
    if (l > 0) nz.push_back(l);
  std::sort(nz.begin(), nz.end());
  bool graded = !nz.empty() && nz.back() > 1.5 * nz[nz.size() / 2];
  if (const char* e = std::getenv("PKRR_PRIO")) graded = std::atoi(e) != 0;
  std::vector<cudaStream_t>& streams = graded ? ctx->work : ctx->work_eq;
  static const bool no_look = std::getenv("PKRR_LOOKAHEAD") && std::atoi(std::getenv("PKRR_LOOKAHEAD")) == 0;
  std::vector<cudaStream_t> look_streams(graded ? ctx->aux : ctx->aux_eq);
  if (no_look) std::fill(look_streams.begin(), look_streams.end(), nullptr);
  std::vector<size_t> sidx(p, 0);
  for (int64_t q : owned) sidx[q] = rank_of[slot[q]];
  std::vector<cudaEvent_t> res_done(p, nullptr);  // residual GEMV of the part's last cell done
  // ---- memory-aware batches of parts (largest first) ----
  auto part_bytes = [&](int64_t q) {
    const int64_t mp = round_up(po.sizes[q], kNB);
    auto qbytes = [&](int64_t cnt) {
      const int64_t qp = round_up(cnt > 0 ? cnt : 1, 64);
      return qp * dp + 2 * qp + qp * mp;
    };
    return 8.0 * static_cast<double>(mp * dp + 12 * mp + 2 * mp * mp + mp * kNB + qbytes(tcount[q]) +
                                     (te ? qbytes(ecount[q]) : 0)) +
           (pk::syrk_ozaki() ? 2.0 * 8.0 * 512.0 * static_cast<double>(mp) : 0.0);
  };
  std::vector<std::vector<int64_t>> batches;
  {
    double need = 0.0;
    for (int64_t q : by_size) need += part_bytes(q);
    double budget = 1e300;
    if (need > 0.4 * ctx->total_mem) {  // only then ask the driver (the query is not free)
      size_t free_b = 0, total_b = 0;
      ck(cudaMemGetInfo(&free_b, &total_b), "meminfo");
      budget = 0.92 * static_cast<double>(free_b + ctx->cached_bytes) - 2.0e9;
    }
    double used = 0.0;
    for (int64_t q : by_size) {
      const double b = part_bytes(q);
      if (batches.empty() || (used + b > budget && !batches.back().empty())) {
        batches.emplace_back();
        used = 0.0;
      }
      batches.back().push_back(q);
      used += b;
    }
  }
  struct Iv {
    cudaEvent_t a, b;
  };
  std::vector<Iv> gram_iv, chol_iv, pred_iv;
  std::vector<cudaEvent_t> part_end(p, nullptr);
  std::vector<std::array<cudaEvent_t, 5>> part_ev(p, std::array<cudaEvent_t, 5>{});
  for (const std::vector<int64_t>& batch : batches) {
    Scope bsc(ctx);  // released (after a device sync) before the next batch
      for (int64_t q : batch) {
      PartBuf& pb = parts[q];
      cudaStream_t ws = streams[sidx[q]];
      ck(cudaStreamWaitEvent(ws, e_pre, 0), "wait");
      part_alloc(bsc, pb, po.sizes[q], d, true, ws);
      part_load(ctx, pb, dX, dy, d, po.order + po.start[q], ws);
      query_alloc(bsc, qt[q], tcount[q], pb.dp, pb.mp);
      if (tcount[q] > 0) {
        pk::launch_gather_rows(dXt, d, tpos[q], tcount[q], qt[q].Xq, qt[q].qp, pb.dp, ws, ctx->counter);
        pk::launch_row_norms(qt[q].Xq, qt[q].qp, pb.dp, pb.dp, qt[q].norms, ws, ctx->counter);
      }
      if (te) {
        query_alloc(bsc, qe[q], ecount[q], pb.dp, pb.mp);
        if (ecount[q] > 0) {
          pk::launch_gather_rows(dXe, d, epos[q], ecount[q], qe[q].Xq, qe[q].qp, pb.dp, ws, ctx->counter);
          pk::launch_row_norms(qe[q].Xq, qe[q].qp, pb.dp, pb.dp, qe[q].norms, ws, ctx->counter);
        }
      }
    }
    hmark("part buffers allocated + loads enqueued");
    // Each part flows gram -> (assemble -> Cholesky -> solves -> predict) per cell on
    // its own prioritised stream, with no cross-part joins: a small part's gram or
    // solves overlap the large part's Cholesky.  Phase times are the UNION of the
    // per-(part, cell) intervals, from events on the launching streams.
    auto ev_on = [&](cudaStream_t st) {
      cudaEvent_t e = ctx->pool_event();
      ck(cudaEventRecord(e, st), "event");
      return e;
    };
    {
      cudaEvent_t f = ev_on(s);
      for (int64_t q : batch) ck(cudaStreamWaitEvent(streams[sidx[q]], f, 0), "wait");
    }
    // enqueue round-robin over (cell, part) so every stream's launch queue fills
    // evenly (a deep queue on one stream would block the host and starve others)
    for (int64_t si = 0; si < ns; ++si) {
      const double sigma = a->sigmas[si];
      for (int64_t q : batch) {  // largest part first
        PartBuf& pb = parts[q];
        cudaStream_t ws = streams[sidx[q]];
        const double m = static_cast<double>(pb.m);
        if (res_done[q]) ck(cudaStreamWaitEvent(ws, res_done[q], 0), "wait");  // K is rewritten
        cudaEvent_t g0 = ev_on(ws);
        // PKRR_DF_GRAM=1: a lone system on the dataflow path forms K and A inside its
        // factorization (first lambda of each sigma; pk::GramFuse) -- measured slower
        // than the gram + assemble kernels at C0 (DF kernel +270 us vs 145 us saved)
        // the first lambda's system A = K + lambda m I leaves the gram's epilogue with K
        if (!(p == 1 && df_gram_fused() && pk::potrf_df_eligible(pb.mp, true)))
          pb.assembled = pk::launch_gram_sym(pb.tmX, pb.norms, pb.mp, pb.dp, pb.m, sigma, pb.K, pb.mp, nullptr, ws,
                                             ctx->counter, false, pb.A, a->lambdas[0] * m);
        f_gram += static_cast<double>(d) * m * (m + 1);
        gram_iv.push_back({g0, ev_on(ws)});
        if (si == 0) part_ev[q][0] = g0, part_ev[q][1] = gram_iv.back().b;
      }
      for (int64_t li = 0; li < nl; ++li) {
        const int64_t cell = li * ns + si;
        const double lambda = a->lambdas[li];
        for (int64_t q : batch) {
          PartBuf& pb = parts[q];
          cudaStream_t ws = streams[sidx[q]];
          const double m = static_cast<double>(pb.m);
          const double shift = lambda * m;
          int* st = dstatus + (cell * p + q) * 2;
          double* rs = dres + (cell * p + q) * 4;
          cudaEvent_t c0 = ev_on(ws);
          const bool gram_fused = li == 0 && p == 1 && df_gram_fused() && pk::potrf_df_eligible(pb.mp, true);
          const pk::GramFuse gf{pb.tmX, pb.norms, pb.K, pb.dp, pb.m, sigma, shift};
          if (!gram_fused && !(li == 0 && pb.assembled))
            pk::launch_assemble(pb.K, pb.A, pb.mp, shift, st, ws, ctx->counter, true);
          const pk::FwdSolve fs{pb.yp, pb.w, pb.z};
          // rank-independent schedule (p == 1): the same at any world size
          const bool fused = pk::launch_potrf(pb.A, pb.tmA, pb.tmLinv, pb.Linv, pb.mp, pb.m, st, ws, ctx->counter,
                                              pb.slices, pb.exps, look_streams[sidx[q]], p == 1, &fs,
                                              gram_fused ? &gf : nullptr);
          cudaEvent_t c1 = ev_on(ws);
          chol_iv.push_back({c0, c1});
          if (li == 0 && si == 0) part_end[q] = c1, part_ev[q][2] = c0, part_ev[q][3] = c1;
          f_chol += chol_flops(pb.m);
          if (res_done[q]) ck(cudaStreamWaitEvent(ws, res_done[q], 0), "wait");  // alpha is rewritten
          if (fused)
            pk::launch_trsv_bwd(pb.A, pb.Linv, pb.mp, pb.z, pb.alpha, pb.scratch, st, ws, ctx->counter);
          else
            pk::launch_trsv(pb.A, pb.Linv, pb.mp, pb.yp, pb.z, pb.alpha, pb.scratch, st, ws, ctx->counter);
          // the residual GEMV (strategies.cpp:310-320) only feeds the reported residual:
          // on the part's idle lookahead stream, overlapping the predictions
          cudaStream_t rst = look_streams[sidx[q]] ? look_streams[sidx[q]] : ws;
          if (rst != ws) ck(cudaStreamWaitEvent(rst, ev_on(ws), 0), "wait");
          pk::launch_symv_lower(pb.K, pb.mp, pb.alpha, pb.Ka, st, rst, ctx->counter);
          pk::launch_residual_finish(pb.Ka, pb.alpha, pb.yp, pb.m, shift, rs, st, rst, ctx->counter);
          if (rst != ws) res_done[q] = ev_on(rst);
          f_other += 4.0 * m * m;
          if (tcount[q] > 0) {
            pk::launch_predict_fused(qt[q].tmQ, pb.tmX, qt[q].norms, pb.norms, qt[q].qp, tcount[q], pb.mp, pb.m,
                                     pb.dp, sigma, pb.alpha, qt[q].partial, qt[q].pred, st, ws, ctx->counter);
            double* dst = pred_t + (cell * pp_parts + (pp_parts > 1 ? q : 0)) * t;
            pk::launch_sse_scatter(qt[q].pred, tpos[q], tcount[q], dyt, dst, rs + 2, st, ws, ctx->counter);
            f_other += 2.0 * tcount[q] * m * (d + 1);
          }
          if (te && ecount[q] > 0) {
            pk::launch_predict_fused(qe[q].tmQ, pb.tmX, qe[q].norms, pb.norms, qe[q].qp, ecount[q], pb.mp, pb.m,
                                     pb.dp, sigma, pb.alpha, qe[q].partial, qe[q].pred, st, ws, ctx->counter);
            double* dst = pred_e + (cell * pp_parts + (pp_parts > 1 ? q : 0)) * te;
            pk::launch_sse_scatter(qe[q].pred, epos[q], ecount[q], dye, dst, rs + 3, st, ws, ctx->counter);
            f_other += 2.0 * ecount[q] * m * (d + 1);
          }
          pred_iv.push_back({c1, ev_on(ws)});
          if (li == 0 && si == 0) part_ev[q][4] = pred_iv.back().b;
        }
      }
    }
    for (int64_t q : batch) {
      cudaEvent_t e = ev_on(streams[sidx[q]]);
      ck(cudaStreamWaitEvent(s, e, 0), "wait");
      if (res_done[q]) ck(cudaStreamWaitEvent(s, res_done[q], 0), "wait");
    }
    if (world == 1 && &batch == &batches.back()) {
      // every cell's combine + reference-order MSE, behind the last batch's parts and
      // before the batch scope synchronises: the host reads statuses, residuals and MSEs
      // after one sync (the failed cells are masked on the host afterwards)
      pk::launch_combine_cells(pred_t, pp_parts, t, ncell, predictor, dyt, comb, dmse, s, ctx->counter);
      if (te)
        pk::launch_combine_cells(pred_e, pp_parts, te, ncell, predictor, dye, comb_e, dmse_e, s, ctx->counter);
    }
    hmark("batch enqueued");
  }
  pk::shadow_report();
  // one GPU: every cell's combine + reference-order MSE goes on the stream now, behind
  // the parts, so the host reads statuses, residuals and MSEs after a single sync (the
  // failed cells are masked on the host afterwards) instead of a sync -> launch -> sync
  // round trip at the end of the call
  ck(cudaEventRecord(t_all.b, s), "event");
  hmark("all enqueued");
  ck(cudaDeviceSynchronize(), "grid");
  hmark("device synchronized");
  cudaEventDestroy(e_pre);

  {
    pkrrgpu_ctx::Pending& P = ctx->pending;
    P.on = true;
    P.all_a = t_all.a;
    P.all_b = t_all.b;
    P.part_a = t_part.a;
    P.part_b = t_part.b;
    P.gram.clear();
    P.chol.clear();
    P.pred.clear();
    for (const Iv& v : gram_iv) P.gram.push_back({v.a, v.b});
    for (const Iv& v : chol_iv) P.chol.push_back({v.a, v.b});
    for (const Iv& v : pred_iv) P.pred.push_back({v.a, v.b});
    P.part_end = part_end;
    P.part_ev = part_ev;
  }

  // the call's small results in one D2H pass through the pinned staging buffer (one
  // sync instead of one per array)
  std::vector<int> st(ncell * p * 2);
  std::vector<double> rs(ncell * p * 4), cmse_h(world == 1 ? ncell : 0), cemse_h(world == 1 && te ? ncell : 0);
  {
    const size_t b_st = sizeof(int) * st.size(), b_rs = sizeof(double) * rs.size();
    const size_t b_m = sizeof(double) * cmse_h.size(), b_e = sizeof(double) * cemse_h.size();
    const size_t o_rs = (b_st + 15) / 16 * 16, o_m = o_rs + b_rs, o_e = o_m + b_m;
    if (o_e + b_e <= 64 * 1024) {
      auto* pin = static_cast<unsigned char*>(ctx->pinned);
      ck(cudaMemcpyAsync(pin, dstatus, b_st, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaMemcpyAsync(pin + o_rs, dres, b_rs, cudaMemcpyDeviceToHost, s), "D2H");
      if (b_m) ck(cudaMemcpyAsync(pin + o_m, dmse, b_m, cudaMemcpyDeviceToHost, s), "D2H");
      if (b_e) ck(cudaMemcpyAsync(pin + o_e, dmse_e, b_e, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaStreamSynchronize(s), "sync");
      std::memcpy(st.data(), pin, b_st);
      std::memcpy(rs.data(), pin + o_rs, b_rs);
      if (b_m) std::memcpy(cmse_h.data(), pin + o_m, b_m);
      if (b_e) std::memcpy(cemse_h.data(), pin + o_e, b_e);
    } else {
      st = to_host(dstatus, ncell * p * 2, s);
      rs = to_host(dres, ncell * p * 4, s);
      if (b_m) cmse_h = to_host(dmse, ncell, s);
      if (b_e) cemse_h = to_host(dmse_e, ncell, s);
    }
  }
  hmark("small results read");
  std::vector<uint8_t> pfail(ncell * p, 0);
  for (int64_t c = 0; c < ncell; ++c)
    for (int64_t q : owned) pfail[c * p + q] = st[(c * p + q) * 2] ? 1 : 0;
  if (o->part_failed) std::memcpy(o->part_failed, pfail.data(), ncell * p);
  std::vector<uint8_t> is_mine(p, 0);
  for (int64_t q : owned) is_mine[q] = 1;
  for (int64_t c = 0; c < ncell; ++c)
    for (int64_t q = 0; q < p; ++q) {
      const bool mine = is_mine[q] != 0;
      if (o->part_sse) o->part_sse[c * p + q] = mine ? rs[(c * p + q) * 4 + 2] : 0.0;
      if (o->part_eval_sse) o->part_eval_sse[c * p + q] = mine ? rs[(c * p + q) * 4 + 3] : 0.0;
      if (o->part_residual) o->part_residual[c * p + q] = mine ? rs[(c * p + q) * 4 + 0] : 0.0;
    }
  if (o->part_test_count)
    for (int64_t q = 0; q < p; ++q) o->part_test_count[q] = tcount[q];
  if (o->part_eval_count)
    for (int64_t q = 0; q < p; ++q) o->part_eval_count[q] = ecount[q];
  o->p_effective = p;
  o->flops_chol = f_chol;
  o->flops_gram = f_gram;
  o->flops_other = f_other;
  D2HBatch outb{ctx->pinned, 64 * 1024, s, {}};
  if (o->part_of) outb.add(o->part_of, po.part_of, n);
  if (o->centers && po.centers) outb.add(o->centers, po.centers, p * d);
  if (o->part_sizes)
    for (int64_t q = 0; q < p; ++q) o->part_sizes[q] = po.sizes[q];

  o->best_index = -1;
  o->pred_rows = pp_parts;
  // this rank's predictions (rows / part slices it does not own are zero): the
  // multi-rank caller sums them over ranks (exact: disjoint) and runs pkrrgpu_combine
  if (o->cell_pred) outb.add(o->cell_pred, pred_t, ncell * pp_parts * t);
  if (o->cell_eval_pred && te) outb.add(o->cell_eval_pred, pred_e, ncell * pp_parts * te);
  if (world == 1) {
    std::vector<uint8_t> cfail(ncell, 0);
    std::vector<double> cres(ncell, 0.0);
    for (int64_t c = 0; c < ncell; ++c)
      for (int64_t q = 0; q < p; ++q) {
        if (pfail[c * p + q]) cfail[c] = 1;
        const double r = rs[(c * p + q) * 4 + 0];
        if (!pfail[c * p + q] && r > cres[c]) cres[c] = r;
      }
    // best = first strict minimum over the non-failed cells (strategies.cpp:499-505)
    std::vector<double> cmse = cmse_h, cemse;
    int64_t best = -1;
    for (int64_t c = 0; c < ncell; ++c) {
      if (cfail[c]) {
        cmse[c] = std::numeric_limits<double>::quiet_NaN();
        continue;
      }
      if (best < 0 || cmse[c] < cmse[best]) best = c;
    }
    o->best_index = best;
    if (best >= 0 && o->best_pred) outb.add(o->best_pred, comb + best * t, t);
    if (te) {
      // the eval set's predictions of the cell chosen on the selection set
      cemse = cemse_h;
      for (int64_t c = 0; c < ncell; ++c)
        if (cfail[c]) cemse[c] = std::numeric_limits<double>::quiet_NaN();
      if (o->best_index >= 0 && o->best_eval_pred) outb.add(o->best_eval_pred, comb_e + o->best_index * te, te);
    }
    if (o->cell_mse) std::memcpy(o->cell_mse, cmse.data(), sizeof(double) * ncell);
    if (o->cell_failed) std::memcpy(o->cell_failed, cfail.data(), ncell);
    if (o->cell_residual) std::memcpy(o->cell_residual, cres.data(), sizeof(double) * ncell);
    if (o->cell_eval_mse && te) std::memcpy(o->cell_eval_mse, cemse.data(), sizeof(double) * ncell);
  }
  outb.flush();
  hmark("results copied out");
  API_END
}

int pkrrgpu_grid_search(pkrrgpu_ctx* ctx, int strategy, const double* X_train,
                        const double* y_train, int64_t n, int64_t d, const double* X_test,
                        const double* y_test, int64_t t, int64_t p, const double* lambdas,
                        int64_t n_lambdas, const double* sigmas, int64_t n_sigmas, uint64_t seed,
                        double* cell_mse, uint8_t* cell_failed, double* cell_residual,
                        int64_t* best_index) {
  pkrrgpu_grid_args a{};
  a.strategy = strategy;
  a.X_train = X_train;
  a.y_train = y_train;
  a.n = n;
  a.d = d;
  a.X_test = X_test;
  a.y_test = y_test;
  a.t = t;
  a.p = p;
  a.lambdas = lambdas;
  a.n_lambdas = n_lambdas;
  a.sigmas = sigmas;
  a.n_sigmas = n_sigmas;
  a.seed = seed;
  a.world = 1;
  pkrrgpu_grid_out o{};
  o.cell_mse = cell_mse;
  o.cell_failed = cell_failed;
  o.cell_residual = cell_residual;
  const int rc = pkrrgpu_grid_search_ex(ctx, &a, &o);
  if (best_index) *best_index = o.best_index;
  return rc;
}

}  // extern "C"
