// multi.cu -- one process, several GPUs: a group of engine contexts driven by one host
// thread per GPU (the reference's run_partitions thread pool, runtime.hpp:
// 70-112, becomes one worker per device).  The p independent per-part models shard
// over the devices by LPT on m^3 (pkrrgpu_grid_search_ex rank/world); the k-means
// partition is optionally sharded bit-exactly over the devices with an in-process
// all-gather (peer copies over NVLink, cudaMemcpyPeer); the per-cell predictions of the
// devices are summed (disjoint, exact) and combined once by pkrrgpu_combine.  The
// result is bitwise the one-context result at any device count, and the same device
// may appear twice (two contexts on one GPU: the test configuration of this build).
#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/pkrr_gpu.h"

extern "C" void pkrrgpu_set_last_error_(const char* msg);

namespace {

// Generation barrier that can be aborted: a rank that fails releases every waiter, whose
// all-gather then reports failure instead of waiting forever.
struct Barrier {
  std::mutex mu;
  std::condition_variable cv;
  int n = 0, waiting = 0;
  long gen = 0;
  bool aborted = false;
  bool wait() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const long g = gen;
    if (++waiting == n) {
      waiting = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    return !aborted || gen != g;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

struct Group;

struct RankLink {
  Group* g = nullptr;
  int rank = 0;
};

struct Group {
  std::vector<int> devices;
  std::vector<pkrrgpu_ctx*> ctx;
  std::vector<RankLink> links;
  Barrier bar;
  std::vector<void*> bufs;  // published all-gather buffers, one per rank
};

// pkrrgpu_allgather_fn over peer memory: rank r's slice r of its own buffer is copied into
// slice r of every other rank's buffer (cudaMemcpyPeer: NVLink between GPUs, a device copy
// when both contexts share one GPU).
int peer_allgather(void* user, void* dev_buf, int64_t bytes) {
  auto* l = static_cast<RankLink*>(user);
  Group& g = *l->g;
  const int W = static_cast<int>(g.ctx.size());
  g.bufs[l->rank] = dev_buf;
  if (!g.bar.wait()) return 1;
  for (int r = 0; r < W; ++r) {
    if (r == l->rank) continue;
    char* dst = static_cast<char*>(dev_buf) + static_cast<int64_t>(r) * bytes;
    const char* src = static_cast<const char*>(g.bufs[r]) + static_cast<int64_t>(r) * bytes;
    if (cudaMemcpyPeer(dst, g.devices[l->rank], src, g.devices[r], static_cast<size_t>(bytes)) != cudaSuccess)
      return 2;
  }
  if (!g.bar.wait()) return 1;  // nobody reuses its buffer before every rank has read it
  return 0;
}

}  // namespace

struct pkrrgpu_multi {
  Group g;
};

extern "C" {

int pkrrgpu_multi_create(const int* devices, int n, pkrrgpu_multi** out) {
  if (!out || n < 1) {
    pkrrgpu_set_last_error_("multi_create: need at least one device");
    return PKRRGPU_INVALID;
  }
  auto* m = new pkrrgpu_multi();
  for (int i = 0; i < n; ++i) {
    const int dev = devices ? devices[i] : i;
    pkrrgpu_ctx* c = nullptr;
    const int rc = pkrrgpu_create(dev, &c);
    if (rc != PKRRGPU_OK) {
      for (auto* x : m->g.ctx) pkrrgpu_destroy(x);
      delete m;
      return rc;
    }
    m->g.devices.push_back(dev);
    m->g.ctx.push_back(c);
  }
  // peer access between distinct devices (NVLink / NVSwitch); absent access falls back
  // to the driver's staged copy inside cudaMemcpyPeer
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (m->g.devices[i] == m->g.devices[j]) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, m->g.devices[i], m->g.devices[j]);
      if (ok) {
        cudaSetDevice(m->g.devices[i]);
        if (cudaDeviceEnablePeerAccess(m->g.devices[j], 0) != cudaSuccess) cudaGetLastError();
      }
    }
  m->g.links.resize(n);
  for (int i = 0; i < n; ++i) m->g.links[i] = RankLink{&m->g, i};
  m->g.bufs.assign(n, nullptr);
  *out = m;
  return PKRRGPU_OK;
}

void pkrrgpu_multi_destroy(pkrrgpu_multi* m) {
  if (!m) return;
  for (auto* c : m->g.ctx) pkrrgpu_destroy(c);
  delete m;
}

int pkrrgpu_multi_size(const pkrrgpu_multi* m) { return m ? static_cast<int>(m->g.ctx.size()) : 0; }

// internal (dist.cu)
int pkrrgpu_multi_device_(const pkrrgpu_multi* m, int i) { return m->g.devices[i]; }

pkrrgpu_ctx* pkrrgpu_multi_context(pkrrgpu_multi* m, int i) {
  return (m && i >= 0 && i < static_cast<int>(m->g.ctx.size())) ? m->g.ctx[i] : nullptr;
}

int pkrrgpu_multi_grid_search(pkrrgpu_multi* m, const pkrrgpu_grid_args* a, pkrrgpu_grid_out* o) {
  if (!m || !a || !o) {
    pkrrgpu_set_last_error_("null argument");
    return PKRRGPU_INVALID;
  }
  const int W = static_cast<int>(m->g.ctx.size());
  if (W == 1) {
    pkrrgpu_grid_args a1 = *a;
    a1.rank = 0;
    a1.world = 1;
    a1.allgather = nullptr;
    return pkrrgpu_grid_search_ex(m->g.ctx[0], &a1, o);
  }
  if (a->n_lambdas <= 0 || a->n_sigmas <= 0 || a->p < 0) {
    pkrrgpu_set_last_error_("grid_search: empty grid");
    return PKRRGPU_INVALID;
  }
  const int64_t ncell = a->n_lambdas * a->n_sigmas;
  const int64_t t = a->t, te = (a->X_eval && a->t_eval > 0) ? a->t_eval : 0;
  const int64_t pmax = a->strategy == PKRRGPU_EXACT ? 1 : std::max<int64_t>(a->p, 1);
  // partition sharding: from 4 devices on by default (below that the redundant partition
  // is as fast, tools/partition_scale.py); PKRR_SHARD_PARTITION=0/1 forces it
  bool shard = W >= 4;
  if (const char* e = std::getenv("PKRR_SHARD_PARTITION")) shard = std::atoi(e) != 0;
  m->g.bar.n = W;
  m->g.bar.aborted = false;

  struct RankOut {
    std::vector<double> pred, epred, sse, esse, res;
    std::vector<uint8_t> failed;
    std::vector<int64_t> tcount, ecount, sizes;
    std::vector<int32_t> part_of;
    std::vector<double> centers;
    pkrrgpu_grid_out o{};
    int rc = 0;
    std::string err;
  };
  std::vector<RankOut> ro(W);
  std::vector<std::thread> th;
  for (int r = 0; r < W; ++r) {
    th.emplace_back([&, r] {
      RankOut& x = ro[r];
      const int64_t P = pmax;  // upper bound of pred_rows
      x.pred.assign(ncell * P * t, 0.0);
      x.epred.assign(ncell * P * (te > 0 ? te : 1), 0.0);
      x.sse.assign(ncell * pmax, 0.0);
      x.esse.assign(ncell * pmax, 0.0);
      x.res.assign(ncell * pmax, 0.0);
      x.failed.assign(ncell * pmax, 0);
      x.tcount.assign(pmax, 0);
      x.ecount.assign(pmax, 0);
      x.sizes.assign(pmax, 0);
      x.part_of.assign(r == 0 && o->part_of ? a->n : 0, 0);
      x.centers.assign(r == 0 && o->centers ? pmax * a->d : 0, 0.0);
      pkrrgpu_grid_args ar = *a;
      ar.rank = r;
      ar.world = W;
      ar.allgather = shard ? peer_allgather : nullptr;
      ar.allgather_user = shard ? &m->g.links[r] : nullptr;
      x.o.cell_pred = x.pred.data();
      x.o.cell_eval_pred = te ? x.epred.data() : nullptr;
      x.o.part_sse = x.sse.data();
      x.o.part_eval_sse = x.esse.data();
      x.o.part_residual = x.res.data();
      x.o.part_failed = x.failed.data();
      x.o.part_test_count = x.tcount.data();
      x.o.part_eval_count = x.ecount.data();
      x.o.part_sizes = x.sizes.data();
      if (!x.part_of.empty()) x.o.part_of = x.part_of.data();
      if (!x.centers.empty()) x.o.centers = x.centers.data();
      x.rc = pkrrgpu_grid_search_ex(m->g.ctx[r], &ar, &x.o);
      if (x.rc != PKRRGPU_OK) {
        x.err = pkrrgpu_last_error();
        m->g.bar.abort();
      }
    });
  }
  for (auto& x : th) x.join();
  for (int r = 0; r < W; ++r)
    if (ro[r].rc != PKRRGPU_OK) {
      pkrrgpu_set_last_error_(("device " + std::to_string(m->g.devices[r]) + ": " + ro[r].err).c_str());
      return ro[r].rc;
    }
  // merge: every (cell, part) value comes from exactly one owner (the others hold 0)
  const int64_t p = ro[0].o.p_effective, P = ro[0].o.pred_rows;
  std::vector<double> pred(ncell * P * t, 0.0), epred(te ? ncell * P * te : 0, 0.0);
  std::vector<uint8_t> pfail(ncell * p, 0), cfail(ncell, 0);
  std::vector<double> cres(ncell, 0.0);
  for (int r = 0; r < W; ++r) {
    for (size_t i = 0; i < pred.size(); ++i) pred[i] += ro[r].pred[i];
    for (size_t i = 0; i < epred.size(); ++i) epred[i] += ro[r].epred[i];
    for (int64_t i = 0; i < ncell * p; ++i) pfail[i] |= ro[r].failed[i];
  }
  for (int64_t c = 0; c < ncell; ++c)
    for (int64_t q = 0; q < p; ++q) {
      if (pfail[c * p + q]) cfail[c] = 1;
      double rq = 0.0;
      for (int r = 0; r < W; ++r) rq += ro[r].res[c * p + q];
      if (!pfail[c * p + q] && rq > cres[c]) cres[c] = rq;
    }
  std::vector<double> cmse(ncell), cemse(ncell);
  int64_t best = -1;
  int rc = pkrrgpu_combine(m->g.ctx[0], a->strategy, p, t, ncell, pred.data(), a->y_test, cfail.data(), cmse.data(),
                           &best, o->best_pred);
  if (rc != PKRRGPU_OK) return rc;
  if (te) {
    // eval set: every cell's MSE; the best (selection) cell's combined predictions
    double unused = 0.0;
    int64_t eb = -1;
    rc = pkrrgpu_combine(m->g.ctx[0], a->strategy, p, te, ncell, epred.data(), a->y_eval, cfail.data(), cemse.data(),
                         &eb, nullptr);
    if (rc != PKRRGPU_OK) return rc;
    if (best >= 0 && o->best_eval_pred)
      rc = pkrrgpu_combine(m->g.ctx[0], a->strategy, p, te, 1, epred.data() + best * P * te, a->y_eval, nullptr,
                           &unused, &eb, o->best_eval_pred);
    if (rc != PKRRGPU_OK) return rc;
  }
  o->best_index = best;
  o->p_effective = p;
  o->pred_rows = P;
  if (o->cell_mse) std::memcpy(o->cell_mse, cmse.data(), sizeof(double) * ncell);
  if (o->cell_eval_mse && te) std::memcpy(o->cell_eval_mse, cemse.data(), sizeof(double) * ncell);
  if (o->cell_failed) std::memcpy(o->cell_failed, cfail.data(), ncell);
  if (o->cell_residual) std::memcpy(o->cell_residual, cres.data(), sizeof(double) * ncell);
  if (o->cell_pred) std::memcpy(o->cell_pred, pred.data(), sizeof(double) * pred.size());
  if (o->cell_eval_pred && te) std::memcpy(o->cell_eval_pred, epred.data(), sizeof(double) * epred.size());
  auto merged = [&](const std::vector<double> RankOut::*f, double* dst) {
    if (!dst) return;
    for (int64_t i = 0; i < ncell * p; ++i) {
      double v = 0.0;
      for (int r = 0; r < W; ++r) v += (ro[r].*f)[i];
      dst[i] = v;
    }
  };
  merged(&RankOut::sse, o->part_sse);
  merged(&RankOut::esse, o->part_eval_sse);
  merged(&RankOut::res, o->part_residual);
  if (o->part_failed) std::memcpy(o->part_failed, pfail.data(), ncell * p);
  for (int64_t q = 0; q < p; ++q) {
    if (o->part_test_count) o->part_test_count[q] = ro[0].tcount[q];
    if (o->part_eval_count) o->part_eval_count[q] = ro[0].ecount[q];
    if (o->part_sizes) o->part_sizes[q] = ro[0].sizes[q];
  }
  if (o->part_of) std::memcpy(o->part_of, ro[0].part_of.data(), sizeof(int32_t) * a->n);
  if (o->centers && !ro[0].centers.empty()) std::memcpy(o->centers, ro[0].centers.data(), sizeof(double) * p * a->d);
  o->flops_chol = o->flops_gram = o->flops_other = 0.0;
  for (int r = 0; r < W; ++r) {
    o->flops_chol += ro[r].o.flops_chol;
    o->flops_gram += ro[r].o.flops_gram;
    o->flops_other += ro[r].o.flops_other;
  }
  return PKRRGPU_OK;
}

}  // extern "C"
