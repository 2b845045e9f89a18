// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper over the UNMODIFIED reference library (pkrr_core sources under
// /root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/libpkrr_ref.so).  It lets the Python tests pin the C restatement
// (oracle/pkrr_oracle.c) against the reference itself and lets bench.py time the
// reference CPU path (`--impl reference`, cpu_baseline kind "reference").
// Dense row-major inputs are turned into dense reference Datasets (indices 0..d-1,
// as standardize() emits them, dataset.cpp:183-193).
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "pkrr/clustering.hpp"
#include "pkrr/dataset.hpp"
#include "pkrr/kernel.hpp"
#include "pkrr/rng.hpp"
#include "pkrr/solver.hpp"
#include "pkrr/strategies.hpp"

using namespace pkrr;

namespace {

thread_local std::string g_err;

Dataset dense(const double* X, const double* y, int64_t n, int64_t d) {
  Dataset ds;
  ds.d = static_cast<std::size_t>(d);
  std::vector<int> idx(d);
  for (int64_t j = 0; j < d; ++j) idx[j] = static_cast<int>(j);
  ds.col.reserve(n * d);
  ds.val.reserve(n * d);
  for (int64_t i = 0; i < n; ++i)
    ds.add_row(idx, std::span<const double>(X + i * d, d), y ? y[i] : 0.0);
  ds.d = static_cast<std::size_t>(d);
  return ds;
}

KernelSpec gauss(double sigma) {
  KernelSpec s;
  s.kind = KernelKind::gaussian;
  s.sigma = sigma;
  return s;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_sub_seed(uint64_t seed, const char* tag) { return sub_seed(seed, tag); }

void ref_rng_stream(uint64_t seed, int64_t count, double* normals, uint64_t* belows,
                    uint64_t below_n) {
  Rng a(seed);
  for (int64_t i = 0; i < count; ++i) normals[i] = a.normal();
  Rng b(seed);
  for (int64_t i = 0; i < count; ++i) belows[i] = b.below(below_n);
}

void ref_random_permutation(uint64_t seed, int64_t n, uint64_t* perm) {
  Rng r(seed);
  const auto p = random_permutation(static_cast<std::size_t>(n), r);
  for (int64_t i = 0; i < n; ++i) perm[i] = p[i];
}

int ref_gram_sym(const double* X, int64_t m, int64_t d, double sigma, double* K) {
  try {
    const Dataset ds = dense(X, nullptr, m, d);
    const Matrix G = gram(gauss(sigma), ds, ds);
    std::memcpy(K, G.a.data(), sizeof(double) * m * m);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_gram_cross(const double* A, int64_t na, const double* B, int64_t nb, int64_t d,
                   double sigma, double* K) {
  try {
    const Dataset a = dense(A, nullptr, na, d);
    const Dataset b = dense(B, nullptr, nb, d);
    const Matrix G = gram(gauss(sigma), a, b);
    std::memcpy(K, G.a.data(), sizeof(double) * na * nb);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Returns 0 ok, 2 NPD (pivot written), 1 other error.
int ref_cholesky(const double* A, int64_t m, double* L, int64_t* pivot) {
  try {
    Matrix M(m, m);
    std::memcpy(M.a.data(), A, sizeof(double) * m * m);
    const CholeskyFactor F = cholesky(std::move(M));
    std::memcpy(L, F.L.a.data(), sizeof(double) * m * m);
    return 0;
  } catch (const NotPositiveDefinite& e) {
    if (pivot) *pivot = static_cast<int64_t>(e.pivot);
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void ref_solve_spd(const double* L, int64_t m, const double* b, double* x) {
  CholeskyFactor F;
  F.L = Matrix(m, m);
  std::memcpy(F.L.a.data(), L, sizeof(double) * m * m);
  const auto r = solve_spd(F, std::span<const double>(b, m));
  std::memcpy(x, r.data(), sizeof(double) * m);
}

int ref_train_krr(const double* X, const double* y, int64_t m, int64_t d, double sigma,
                  double lambda, double* alpha, double* residual, int64_t* pivot) {
  try {
    const Dataset ds = dense(X, y, m, d);
    const KrrModel model = train_krr(ds, gauss(sigma), lambda);
    std::memcpy(alpha, model.alpha.data(), sizeof(double) * m);
    if (residual) *residual = model.residual_ratio;
    return 0;
  } catch (const NotPositiveDefinite& e) {
    if (pivot) *pivot = static_cast<int64_t>(e.pivot);
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// KrrModel::predict over q query rows (model trained by train_krr).
int ref_train_predict(const double* X, const double* y, int64_t m, int64_t d, double sigma,
                      double lambda, const double* Q, int64_t q, double* out) {
  try {
    const Dataset ds = dense(X, y, m, d);
    const KrrModel model = train_krr(ds, gauss(sigma), lambda);
    const Dataset qs = dense(Q, nullptr, q, d);
    for (int64_t j = 0; j < q; ++j) out[j] = model.predict(qs.row(j));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

static void copy_clustering(const Clustering& c, int32_t* membership, double* centers,
                            int64_t* sizes, int64_t d) {
  for (std::size_t i = 0; i < c.membership.size(); ++i) membership[i] = c.membership[i];
  for (int j = 0; j < c.k; ++j) {
    std::memcpy(centers + j * d, c.centers[j].data(), sizeof(double) * d);
    sizes[j] = static_cast<int64_t>(c.sizes[j]);
  }
}

int ref_kmeans(const double* X, int64_t n, int64_t d, int k, uint64_t seed, double threshold,
               int max_iters, int32_t* membership, double* centers, int64_t* sizes,
               int* iterations, double* wcss) {
  try {
    const Dataset ds = dense(X, nullptr, n, d);
    KMeansParams p;
    p.threshold = threshold;
    p.max_iters = max_iters;
    KMeansDiag diag;
    const Clustering c = kmeans(ds, k, seed, p, &diag);
    copy_clustering(c, membership, centers, sizes, d);
    if (iterations) *iterations = diag.iterations;
    if (wcss)
      for (std::size_t i = 0; i < diag.wcss.size(); ++i) wcss[i] = diag.wcss[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_kbalance(const double* X, int64_t n, int64_t d, int k, uint64_t seed, double threshold,
                 int max_iters, int recompute, int32_t* membership, double* centers,
                 int64_t* sizes) {
  try {
    const Dataset ds = dense(X, nullptr, n, d);
    KMeansParams p;
    p.threshold = threshold;
    p.max_iters = max_iters;
    p.recompute_centers = recompute != 0;
    const Clustering c = kbalance(ds, k, seed, p);
    copy_clustering(c, membership, centers, sizes, d);
    return 0;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_nearest_center(const double* centers, int k, int64_t d, const double* x) {
  std::vector<std::vector<double>> c(k);
  for (int j = 0; j < k; ++j) c[j].assign(centers + j * d, centers + (j + 1) * d);
  const Dataset q = dense(x, nullptr, 1, d);
  return nearest_center(c, q.row(0));
}

// make_partition: part id per row, centers (p*d) when defined. Returns p or -1.
int64_t ref_make_partition(int kind, const double* X, int64_t n, int64_t d, int64_t p,
                           uint64_t seed, int32_t* part_of, double* centers) {
  try {
    const Dataset ds = dense(X, nullptr, n, d);
    const PartitionSet ps = make_partition(static_cast<StrategyKind>(kind), ds, p, seed);
    for (std::size_t t = 0; t < ps.p; ++t)
      for (std::size_t i : ps.parts[t]) part_of[i] = static_cast<int32_t>(t);
    if (ps.has_centers() && centers)
      for (std::size_t t = 0; t < ps.p; ++t)
        std::memcpy(centers + t * d, ps.centers[t].data(), sizeof(double) * d);
    return static_cast<int64_t>(ps.p);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// grid_search through the reference's public API.  Returns best index, -1 when
// no cell succeeded, -2 on error.
int64_t ref_grid_search(int kind, const double* Xtr, const double* ytr, int64_t n, int64_t d,
                        const double* Xte, const double* yte, int64_t t, int64_t p,
                        const double* lambdas, int64_t nl, const double* sigmas, int64_t ns,
                        uint64_t seed, int64_t workers, double* cell_mse, uint8_t* cell_failed,
                        double* cell_residual) {
  try {
    const Dataset train = dense(Xtr, ytr, n, d);
    const Dataset test = dense(Xte, yte, t, d);
    GridOptions opt;
    opt.workers = static_cast<std::size_t>(workers < 1 ? 1 : workers);
    const GridResult r =
        grid_search(static_cast<StrategyKind>(kind), train, test, p,
                    std::span<const double>(lambdas, nl), std::span<const double>(sigmas, ns),
                    seed, opt);
    for (std::size_t c = 0; c < r.cells.size(); ++c) {
      cell_mse[c] = r.cells[c].mse;
      cell_failed[c] = r.cells[c].failed ? 1 : 0;
      cell_residual[c] = r.cells[c].max_residual;
    }
    return r.has_best() ? static_cast<int64_t>(r.best_index) : -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// train_partitions + predict_nearest (the 4-stage API path, strategies.cpp:104-149)
int ref_train_predict_nearest(int kind, const double* Xtr, const double* ytr, int64_t n,
                              int64_t d, int64_t p, uint64_t seed, double sigma, double lambda,
                              int64_t workers, const double* Q, int64_t q, double* out) {
  try {
    const Dataset train = dense(Xtr, ytr, n, d);
    const PartitionSet ps = make_partition(static_cast<StrategyKind>(kind), train, p, seed);
    const TrainedPartitions tp =
        train_partitions(ps, train, gauss(sigma), lambda, static_cast<std::size_t>(workers));
    const Dataset qs = dense(Q, nullptr, q, d);
    for (int64_t j = 0; j < q; ++j) out[j] = predict_nearest(tp.models, ps.centers, qs.row(j));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The 4-stage API with a caller-given partition (strategies.hpp:50-58): the PartitionSet
// is rebuilt from part_of (rows in train row order, strategies.cpp:97-99), trained by the
// reference's train_partitions(ps, train, spec, lambda, workers), and q query rows are
// predicted by predict_nearest (centers given) or the single model (p == 1, no centers).
// alpha_out: the parts' alphas concatenated in part order (n entries); residual_out[p],
// seconds_out[p] (the per-task wall clocks of run_partitions, runtime.hpp:85-90).
int ref_train_partitions_predict(const double* Xtr, const double* ytr, int64_t n, int64_t d,
                                 const int32_t* part_of, int64_t p, const double* centers,
                                 double sigma, double lambda, int64_t workers, const double* Q,
                                 int64_t q, double* alpha_out, double* residual_out,
                                 double* pred_out, double* seconds_out) {
  try {
    const Dataset train = dense(Xtr, ytr, n, d);
    PartitionSet ps;
    ps.p = static_cast<std::size_t>(p);
    ps.parts.assign(ps.p, {});
    for (int64_t i = 0; i < n; ++i) ps.parts[part_of[i]].push_back(static_cast<std::size_t>(i));
    if (centers)
      for (int64_t t = 0; t < p; ++t) ps.centers.emplace_back(centers + t * d, centers + (t + 1) * d);
    const TrainedPartitions tp =
        train_partitions(ps, train, gauss(sigma), lambda, static_cast<std::size_t>(workers < 1 ? 1 : workers));
    int64_t at = 0;
    for (int64_t t = 0; t < p; ++t) {
      const auto& a = tp.models[t].alpha;
      std::memcpy(alpha_out + at, a.data(), sizeof(double) * a.size());
      at += static_cast<int64_t>(a.size());
      if (residual_out) residual_out[t] = tp.models[t].residual_ratio;
      if (seconds_out) seconds_out[t] = tp.stats.per_task[t].wall_seconds;
    }
    const Dataset qs = dense(Q, nullptr, q, d);
    for (int64_t j = 0; j < q; ++j)
      pred_out[j] = centers ? predict_nearest(tp.models, ps.centers, qs.row(j))
                            : tp.models[0].predict(qs.row(j));
    return 0;
  } catch (const NotPositiveDefinite& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// dataset.cpp:199-232 through the reference's own standardize (dense rows in)
int ref_standardize(const double* Xtr, int64_t n, int64_t d, const double* Xte, int64_t t, double* Xtr_out,
                    double* Xte_out, double* mean, double* stddev) {
  try {
    const Dataset tr = dense(Xtr, nullptr, n, d);
    const Dataset te = t > 0 ? dense(Xte, nullptr, t, d) : Dataset{};
    const StandardizeResult r = standardize(tr, te);
    for (int64_t i = 0; i < n; ++i) {
      const SparseRow row = r.train.row(i);
      for (std::size_t k = 0; k < row.nnz(); ++k) Xtr_out[i * d + row.idx[k]] = row.val[k];
    }
    for (int64_t i = 0; i < t; ++i) {
      const SparseRow row = r.test.row(i);
      for (std::size_t k = 0; k < row.nnz(); ++k) Xte_out[i * d + row.idx[k]] = row.val[k];
    }
    for (int64_t j = 0; j < d; ++j) {
      mean[j] = r.stats.mean[j];
      stddev[j] = r.stats.stddev[j];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// strategies.cpp:204-234
int ref_auto_sigma_grid(const double* X, int64_t n, int64_t d, uint64_t seed, double* grid9) {
  try {
    const Dataset tr = dense(X, nullptr, n, d);
    const std::vector<double> g = auto_sigma_grid(tr, seed);
    for (std::size_t i = 0; i < g.size() && i < 9; ++i) grid9[i] = g[i];
    return static_cast<int>(g.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// dataset.cpp:83-125 through the reference's own loader; two calls: sizes, then arrays
int ref_load_libsvm(const char* path, int64_t* n, int64_t* d, int64_t* nnz, int64_t* row_ptr, int32_t* col,
                    double* val, double* y) {
  try {
    const Dataset ds = load_libsvm(path);
    *n = static_cast<int64_t>(ds.n);
    *d = static_cast<int64_t>(ds.d);
    *nnz = static_cast<int64_t>(ds.col.size());
    if (row_ptr)
      for (std::size_t i = 0; i < ds.row_ptr.size(); ++i) row_ptr[i] = static_cast<int64_t>(ds.row_ptr[i]);
    if (col)
      for (std::size_t i = 0; i < ds.col.size(); ++i) col[i] = ds.col[i];
    if (val) std::memcpy(val, ds.val.data(), sizeof(double) * ds.val.size());
    if (y) std::memcpy(y, ds.y.data(), sizeof(double) * ds.y.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
