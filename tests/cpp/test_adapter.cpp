// C++ parity test of include/pkrr_gpu.hpp (pkrr::gpu::*) against the reference
// library itself (pkrr::*, linked from oracle/_ref/libpkrr_ref.so).  Built in the
// build container (needs /root/reference headers); run on the GPU box by
// tests/test_gpu_adapter.py.  Exit status 0 iff every check passes.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <vector>

#include "pkrr/rng.hpp"
#include "pkrr_gpu.hpp"

using namespace pkrr;

static int g_fail = 0;
#define CHECK(cond, what)                                              \
  do {                                                                 \
    const bool ok_ = (cond);                                           \
    std::printf("[%s] %s\n", ok_ ? "PASS" : "FAIL", what);            \
    if (!ok_) ++g_fail;                                                \
  } while (0)

static Dataset mixture(std::size_t n, std::size_t d, std::size_t comps, std::uint64_t seed) {
  Rng rng(seed);
  std::vector<std::vector<double>> means(comps, std::vector<double>(d));
  for (auto& m : means)
    for (auto& v : m) v = 3.0 * rng.normal();
  Dataset ds;
  ds.d = d;
  std::vector<int> idx(d);
  for (std::size_t j = 0; j < d; ++j) idx[j] = static_cast<int>(j);
  std::vector<double> x(d);
  for (std::size_t i = 0; i < n; ++i) {
    const auto& m = means[rng.below(comps)];
    for (std::size_t j = 0; j < d; ++j) x[j] = m[j] + rng.normal();
    ds.add_row(idx, x, std::sin(x[0]) + 0.1 * rng.normal());
  }
  ds.d = d;
  return ds;
}

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num) / std::max(std::sqrt(den), 1e-300);
}

int main() {
  const Dataset X = mixture(700, 12, 5, 3);
  KernelSpec spec;
  spec.sigma = 2.5;
  // gram
  {
    OpCount a, b;
    const Matrix G = gpu::gram(spec, X, X, &a);
    const Matrix R = pkrr::gram(spec, X, X, &b);
    double worst = 0;
    bool sym = true;
    for (std::size_t i = 0; i < G.rows; ++i)
      for (std::size_t j = 0; j < G.cols; ++j) {
        worst = std::max(worst, std::fabs(G(i, j) - R(i, j)));
        sym = sym && G(i, j) == G(j, i);
      }
    CHECK(worst <= 1e-13 && sym, "gram: |K_gpu - K_ref| <= 1e-13, bitwise symmetric");
    CHECK(a.gram_flops == b.gram_flops, "gram: OpCount.gram_flops identical");
  }
  // cholesky + NPD
  {
    Matrix A = pkrr::assemble_system(pkrr::gram(spec, X, X), 1e-3, X.n);
    const CholeskyFactor F = gpu::cholesky(A);
    const CholeskyFactor R = pkrr::cholesky(A);
    CHECK(rel(F.L.a, R.L.a) <= 1e-12, "cholesky: rel ||L_gpu - L_ref|| <= 1e-12");
    Matrix B(3, 3);
    B(0, 0) = 1;
    B(1, 1) = -1;
    B(2, 2) = 1;
    bool threw = false;
    try {
      gpu::cholesky(B);
      std::printf("  no exception\n");
    } catch (const NotPositiveDefinite& e) {
      threw = e.pivot == 1;
      std::printf("  NotPositiveDefinite pivot=%zu\n", e.pivot);
    } catch (const std::exception& e) {
      std::printf("  other exception: %s\n", e.what());
    }
    CHECK(threw, "cholesky: indefinite -> NotPositiveDefinite(pivot 1)");
    std::vector<double> y(X.y.begin(), X.y.end());
    CHECK(rel(gpu::solve_spd(F, y), pkrr::solve_spd(R, y)) <= 1e-10, "solve_spd: rel <= 1e-10");
  }
  // train_krr
  {
    OpCount a, b;
    const KrrModel g = gpu::train_krr(X, spec, 1e-4, &a);
    const KrrModel r = pkrr::train_krr(X, spec, 1e-4, &b);
    CHECK(rel(g.alpha, r.alpha) <= 1e-8, "train_krr: rel ||alpha_gpu - alpha_ref|| <= 1e-8");
    CHECK(g.residual_ratio <= 1e-8, "train_krr: residual <= 1e-8");
    CHECK(a.gram_flops == b.gram_flops && a.solve_flops == b.solve_flops, "train_krr: OpCount identical");
    // the returned model predicts with the reference's own KrrModel::predict
    CHECK(std::fabs(g.predict(X.row(5)) - r.predict(X.row(5))) <= 1e-8 * std::fabs(r.predict(X.row(5))) + 1e-12,
          "train_krr: KrrModel::predict agrees");
  }
  // clustering
  {
    const Clustering g = gpu::kmeans(X, 6, 9), r = pkrr::kmeans(X, 6, 9);
    CHECK(g.membership == r.membership && g.centers == r.centers && g.sizes == r.sizes,
          "kmeans: membership, centers, sizes bitwise");
    const Clustering gb = gpu::kbalance(X, 6, 9), rb = pkrr::kbalance(X, 6, 9);
    CHECK(gb.membership == rb.membership && gb.centers == rb.centers, "kbalance: bitwise");
    bool near = true;
    for (std::size_t i = 0; i < 50; ++i)
      near = near && gpu::nearest_center(r.centers, X.row(i)) == pkrr::nearest_center(r.centers, X.row(i));
    CHECK(near, "nearest_center: identical");
    for (StrategyKind k : {StrategyKind::exact, StrategyKind::dc, StrategyKind::kk2, StrategyKind::bk2}) {
      const PartitionSet a = gpu::make_partition(k, X, 4, 21), b = pkrr::make_partition(k, X, 4, 21);
      CHECK(a.p == b.p && a.parts == b.parts && a.centers == b.centers, "make_partition: identical parts/centers");
    }
  }
  // train_partitions
  {
    const PartitionSet ps = pkrr::make_partition(StrategyKind::kk2, X, 3, 5);
    const TrainedPartitions g = gpu::train_partitions(ps, X, spec, 1e-3);
    const TrainedPartitions r = pkrr::train_partitions(ps, X, spec, 1e-3);
    bool ok = true;
    for (std::size_t t = 0; t < 3; ++t) ok = ok && rel(g.models[t].alpha, r.models[t].alpha) <= 1e-8;
    CHECK(ok, "train_partitions: per-part alpha rel <= 1e-8");
    const Dataset Q = mixture(40, 12, 5, 7);
    bool pn = true;
    for (std::size_t j = 0; j < Q.n; ++j) {
      const double a = pkrr::predict_nearest(g.models, ps.centers, Q.row(j));
      const double b = pkrr::predict_nearest(r.models, ps.centers, Q.row(j));
      pn = pn && std::fabs(a - b) <= 1e-8 * std::fabs(b) + 1e-12;
    }
    CHECK(pn, "predict_nearest over GPU-trained models agrees");
  }
  // train_partitions with the caller's PartitionSet (random partition: rows in permutation
  // order), GPU predict stage vs the reference's predict_nearest / predict_average /
  // predict_oracle (strategies.cpp:135-166)
  {
    const Dataset Q = mixture(60, 12, 5, 8);
    for (StrategyKind k : {StrategyKind::kk2, StrategyKind::dc, StrategyKind::bk2}) {
      const PartitionSet ps = pkrr::make_partition(k, X, 4, 13);
      const TrainedPartitions g = gpu::train_partitions(ps, X, spec, 1e-3);
      const TrainedPartitions r = pkrr::train_partitions(ps, X, spec, 1e-3);
      bool ok = g.models.size() == r.models.size();
      for (std::size_t t = 0; ok && t < r.models.size(); ++t)
        ok = rel(g.models[t].alpha, r.models[t].alpha) <= 1e-8 && g.models[t].support.val == r.models[t].support.val &&
             g.models[t].train_ops.solve_flops == r.models[t].train_ops.solve_flops;
      std::string what = std::string("train_partitions(") + strategy_name(k) + "): alpha rel <= 1e-8, same supports";
      CHECK(ok, what.c_str());
      // batched GPU predict over the GPU-resident models, and over the host models
      const gpu::DeviceModels dm = gpu::train_partitions_device(ps, X, spec, 1e-3);
      std::vector<double> ref_avg(Q.n), ref_or(Q.n);
      std::vector<std::size_t> ref_or_t(Q.n);
      OpCount oa, ob;
      for (std::size_t j = 0; j < Q.n; ++j) {
        ref_avg[j] = pkrr::predict_average(r.models, Q.row(j), &ob);
        const auto pr = pkrr::predict_oracle(r.models, Q.row(j), Q.y[j]);
        ref_or[j] = pr.first;
        ref_or_t[j] = pr.second;
      }
      const std::vector<double> avg = gpu::predict_average(g.models, Q, &oa);
      CHECK(rel(avg, ref_avg) <= 1e-8 && oa.predict_flops == ob.predict_flops,
            "predict_average: GPU batched vs reference per row, rel <= 1e-8, OpCount identical");
      const auto orc = gpu::predict_oracle(g.models, Q);
      bool oc = true;
      std::vector<double> orv;
      for (std::size_t j = 0; j < Q.n; ++j) orv.push_back(orc[j].first), oc = oc && orc[j].second == ref_or_t[j];
      CHECK(oc && rel(orv, ref_or) <= 1e-8, "predict_oracle: same chosen models, rel <= 1e-8");
      for (std::size_t t = 0; t < ps.p; ++t) {
        std::vector<double> want(Q.n);
        for (std::size_t j = 0; j < Q.n; ++j) want[j] = r.models[t].predict(Q.row(j));
        CHECK(rel(gpu::predict(dm, t, Q), want) <= 1e-8, "KrrModel::predict batched on device models, rel <= 1e-8");
      }
      if (!ps.has_centers()) continue;
      std::vector<double> want(Q.n);
      OpCount rc_ops, gc_ops;
      for (std::size_t j = 0; j < Q.n; ++j) want[j] = pkrr::predict_nearest(r.models, ps.centers, Q.row(j), &rc_ops);
      CHECK(rel(gpu::predict_nearest(dm, Q), want) <= 1e-8, "predict_nearest: device models vs reference, rel <= 1e-8");
      CHECK(rel(gpu::predict_nearest(g.models, ps.centers, Q, &gc_ops), want) <= 1e-8 &&
                gc_ops.predict_flops == rc_ops.predict_flops,
            "predict_nearest: host models batched on the GPU, rel <= 1e-8, OpCount identical");
      const double one = gpu::predict_nearest(std::span<const KrrModel>(g.models), ps.centers, Q.row(3));
      CHECK(std::fabs(one - want[3]) <= 1e-8 * std::fabs(want[3]) + 1e-12, "predict_nearest: drop-in single row");
    }
  }
  // a failed kernel launch is reported, never OK with garbage (PKRR_FAULT_LAUNCH test hook)
  {
    setenv("PKRR_FAULT_LAUNCH", "3", 1);
    pkrrgpu_ctx* c = nullptr;
    const int rc0 = pkrrgpu_create(0, &c);
    unsetenv("PKRR_FAULT_LAUNCH");
    std::vector<double> Xd = gpu::detail::dense(X), alpha(X.n);
    double res = 0;
    int64_t piv = -1;
    const int rc = rc0 == PKRRGPU_OK ? pkrrgpu_train_krr(c, Xd.data(), X.y.data(), X.n, X.d, 2.5, 1e-4,
                                                         alpha.data(), &res, &piv)
                                     : rc0;
    const std::string msg = pkrrgpu_last_error();
    std::printf("  forced bad launch: rc=%d \"%s\"\n", rc, msg.c_str());
    CHECK(rc == PKRRGPU_CUDA && msg.find("launch") != std::string::npos, "forced bad launch -> PKRRGPU_CUDA");
    const int rc2 = pkrrgpu_train_krr(c, Xd.data(), X.y.data(), X.n, X.d, 2.5, 1e-4, alpha.data(), &res, &piv);
    CHECK(rc2 == PKRRGPU_OK, "the context recovers: the next call (no fault) is OK");
    pkrrgpu_destroy(c);
  }
  // two contexts on one GPU (one host thread each) == one context, bitwise; the sharded
  // partition's peer all-gather included
  {
    setenv("PKRR_SHARD_PARTITION", "1", 1);
    gpu::Group two({0, 0});
    const Dataset tr = mixture(2400, 10, 6, 41), te = mixture(300, 10, 6, 42);
    const std::vector<double> lam{1e-4, 1e-2}, sig{1.5, 4.0};
    for (StrategyKind k : {StrategyKind::kk2, StrategyKind::bk2, StrategyKind::kk, StrategyKind::kk3,
                           StrategyKind::dc, StrategyKind::exact}) {
      const GridResult a = gpu::grid_search(k, tr, te, 6, lam, sig, 9);
      const GridResult b = gpu::grid_search(k, tr, te, 6, lam, sig, 9, GridOptions{}, two);
      bool same = a.best_index == b.best_index && a.cells.size() == b.cells.size();
      for (std::size_t c = 0; same && c < a.cells.size(); ++c)
        same = std::memcmp(&a.cells[c].mse, &b.cells[c].mse, sizeof(double)) == 0 &&
               a.cells[c].failed == b.cells[c].failed && a.cells[c].max_residual == b.cells[c].max_residual &&
               a.cells[c].flops == b.cells[c].flops;
      std::string what = std::string("grid_search ") + strategy_name(k) + ": 2 contexts on one GPU == 1, bitwise";
      CHECK(same, what.c_str());
    }
    unsetenv("PKRR_SHARD_PARTITION");
  }
  // grid_search
  {
    const Dataset tr = mixture(1600, 10, 6, 11), te = mixture(300, 10, 6, 12);
    const std::vector<double> lam{1e-4, 1e-2}, sig{1.5, 4.0};
    for (StrategyKind k : {StrategyKind::exact, StrategyKind::dc, StrategyKind::kk, StrategyKind::kk2,
                           StrategyKind::kk3, StrategyKind::bk, StrategyKind::bk2, StrategyKind::bk3}) {
      const GridResult g = gpu::grid_search(k, tr, te, 4, lam, sig, 7);
      const GridResult r = pkrr::grid_search(k, tr, te, 4, lam, sig, 7);
      bool ok = g.cells.size() == r.cells.size() && g.best_index == r.best_index;
      bool counters = true;
      for (std::size_t c = 0; ok && c < g.cells.size(); ++c) {
        ok = ok && g.cells[c].failed == r.cells[c].failed &&
             std::fabs(g.cells[c].mse - r.cells[c].mse) <= 1e-8 * std::fabs(r.cells[c].mse);
        counters = counters && g.cells[c].flops == r.cells[c].flops && g.cells[c].messages == r.cells[c].messages &&
                   g.cells[c].bytes == r.cells[c].bytes && g.cells[c].modeled_seconds == r.cells[c].modeled_seconds;
      }
      std::string what = std::string("grid_search ") + strategy_name(k) + ": mse rel <= 1e-8, same best cell";
      CHECK(ok, what.c_str());
      what = std::string("grid_search ") + strategy_name(k) + ": flops/messages/bytes/modeled_seconds identical";
      CHECK(counters, what.c_str());
    }
  }
  // standardize / auto_sigma_grid (dataset.cpp:199-232, strategies.cpp:204-234): bitwise
  {
    const Dataset tr = mixture(900, 7, 4, 21), te = mixture(120, 7, 4, 22);
    const StandardizeResult g = gpu::standardize(tr, te);
    const StandardizeResult r = pkrr::standardize(tr, te);
    CHECK(g.stats.mean == r.stats.mean && g.stats.stddev == r.stats.stddev, "standardize: mean/stddev bitwise");
    CHECK(g.train.val == r.train.val && g.train.col == r.train.col && g.train.row_ptr == r.train.row_ptr &&
              g.train.y == r.train.y && g.test.val == r.test.val && g.test.d == r.test.d,
          "standardize: train/test rows bitwise");
    CHECK(gpu::auto_sigma_grid(tr, 5) == pkrr::auto_sigma_grid(tr, 5), "auto_sigma_grid bitwise (n <= 512)");
    const Dataset big = mixture(3000, 9, 6, 23);
    CHECK(gpu::auto_sigma_grid(big, 77) == pkrr::auto_sigma_grid(big, 77), "auto_sigma_grid bitwise (n > 512)");
    bool threw = false;
    try {
      gpu::standardize(Dataset{}, te);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw, "standardize: empty training set -> invalid_argument");
  }
  // load_libsvm (dataset.cpp:83-125): the same Dataset, bitwise
  {
    const Dataset src = mixture(5000, 11, 4, 31);
    const std::string path = "/tmp/pkrr_adapter_test.svm";
    save_libsvm(src, path);
    const Dataset g = gpu::load_libsvm(path);
    const Dataset r = pkrr::load_libsvm(path);
    CHECK(g.n == r.n && g.d == r.d && g.row_ptr == r.row_ptr && g.col == r.col && g.val == r.val && g.y == r.y,
          "load_libsvm: identical Dataset");
    bool threw = false;
    try {
      gpu::load_libsvm("/nonexistent.svm");
    } catch (const std::runtime_error&) {
      threw = true;
    }
    CHECK(threw, "load_libsvm: missing file -> runtime_error");
  }
  std::printf("%d failure(s)\n", g_fail);
  return g_fail ? 1 : 0;
}
