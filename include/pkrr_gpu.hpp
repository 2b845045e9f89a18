// pkrr_gpu.hpp -- header-only C++ adapter: the reference library's hot-path API
// (proj/include/pkrr/{kernel,solver,clustering,strategies}.hpp) re-exposed over
// the B200 engine's C ABI (pkrr_gpu.h).  Same types, same signatures, same
// exceptions, in namespace pkrr::gpu, so a caller switches with a using-
// declaration or a namespace prefix:
//
//   Matrix        gram(spec, A, B, ops)                     kernel.hpp:40
//   Matrix        assemble_system(K, lambda, m)             kernel.hpp:44
//   CholeskyFactor cholesky(A, ops)                         solver.hpp:29
//   vector<double> solve_spd(F, b, ops)                     solver.hpp:32-33
//   KrrModel      train_krr(data, spec, lambda, ops)        solver.hpp:52-53
//   Clustering    kmeans / kbalance                         clustering.hpp:33-41
//   int           nearest_center(centers, x)                clustering.hpp:44-45
//   PartitionSet  make_partition(kind, train, p, seed)      strategies.hpp:40-41
//   TrainedPartitions train_partitions(ps, train, spec, lambda, workers)  :50-52
//   GridResult    grid_search(kind, train, test, p, lambdas, sigmas, seed, options)  :117-120
//
// The analytic OpCount charges follow the reference accounting exactly
// (kernel.cpp:68-79, solver.cpp:39-42/67-70, strategies.cpp:285-329/420-452), so
// counters, messages, bytes and modeled_seconds in GridResult are identical.
// Requires the reference headers on the include path and libpkrr_gpu.so at link.
#pragma once

#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "pkrr/clustering.hpp"
#include "pkrr/dataset.hpp"
#include "pkrr/kernel.hpp"
#include "pkrr/runtime.hpp"
#include "pkrr/solver.hpp"
#include "pkrr/strategies.hpp"
#include "pkrr_gpu.h"

namespace pkrr::gpu {

// ---- engine handle (one per device; the default engine uses device 0) -------
class Engine {
 public:
  explicit Engine(int device = 0) {
    if (pkrrgpu_create(device, &ctx_) != PKRRGPU_OK)
      throw std::runtime_error(std::string("pkrr-gpu: ") + pkrrgpu_last_error());
  }
  ~Engine() { pkrrgpu_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  pkrrgpu_ctx* get() const { return ctx_; }

 private:
  pkrrgpu_ctx* ctx_ = nullptr;
};

inline Engine& default_engine() {
  static Engine e(0);
  return e;
}

namespace detail {

// rethrow the reference's exception type for a C-ABI status
inline void check(int rc, int64_t pivot = -1) {
  if (rc == PKRRGPU_OK) return;
  const std::string msg = pkrrgpu_last_error();
  if (rc == PKRRGPU_NPD) throw NotPositiveDefinite(static_cast<std::size_t>(pivot < 0 ? 0 : pivot), 0.0);
  if (rc == PKRRGPU_INVALID) throw std::invalid_argument(msg);
  if (rc == PKRRGPU_LOGIC) throw std::logic_error(msg);
  throw std::runtime_error("pkrr-gpu: " + msg);
}

// dense row-major copy of a (possibly sparse) dataset, d columns
inline std::vector<double> dense(const Dataset& ds) {
  std::vector<double> X(ds.n * ds.d, 0.0);
  for (std::size_t i = 0; i < ds.n; ++i) {
    const SparseRow r = ds.row(i);
    for (std::size_t k = 0; k < r.nnz(); ++k) X[i * ds.d + r.idx[k]] = r.val[k];
  }
  return X;
}

inline std::uint64_t gauss_pair_flops(std::size_t nnz_a, std::size_t nnz_b) {
  return kernel_eval_flops(KernelSpec{}, nnz_a, nnz_b);  // gaussian: 2*min(nnz) + 6
}

inline void require_gaussian(const KernelSpec& spec) {
  if (spec.kind != KernelKind::gaussian)
    throw std::invalid_argument("pkrr-gpu: only the gaussian kernel is on the GPU path");
  if (!(spec.sigma > 0.0)) throw std::invalid_argument("gaussian kernel needs sigma > 0");
}

}  // namespace detail

// ---- kernel.hpp --------------------------------------------------------------
inline Matrix gram(const KernelSpec& spec, const Dataset& A, const Dataset& B, OpCount* ops = nullptr) {
  detail::require_gaussian(spec);
  if (A.d != B.d) throw std::invalid_argument("gram: dimension mismatch");
  Matrix K(A.n, B.n);
  const std::vector<double> XA = detail::dense(A);
  if (&A == &B) {
    detail::check(pkrrgpu_gram(default_engine().get(), XA.data(), A.n, XA.data(), A.n, A.d, spec.sigma,
                               K.a.data()));
  } else {
    const std::vector<double> XB = detail::dense(B);
    detail::check(pkrrgpu_gram(default_engine().get(), XA.data(), A.n, XB.data(), B.n, A.d, spec.sigma,
                               K.a.data()));
  }
  if (ops) {  // kernel.cpp:90-131 charges
    std::uint64_t f = 0;
    for (std::size_t i = 0; i < A.n; ++i) f += 2 * A.row(i).nnz();
    if (&A != &B)
      for (std::size_t j = 0; j < B.n; ++j) f += 2 * B.row(j).nnz();
    for (std::size_t i = 0; i < A.n; ++i)
      for (std::size_t j = (&A == &B ? i : 0); j < B.n; ++j)
        f += detail::gauss_pair_flops(A.row(i).nnz(), B.row(j).nnz());
    ops->gram_flops += f;
  }
  return K;
}

inline Matrix assemble_system(const Matrix& K, double lambda, std::size_t m) {
  if (K.rows != K.cols) throw std::invalid_argument("assemble_system: matrix not square");
  if (!(lambda > 0.0)) throw std::invalid_argument("assemble_system: lambda must be > 0");
  Matrix A(K.rows, K.cols);
  detail::check(pkrrgpu_assemble(default_engine().get(), K.a.data(), K.rows, lambda, m, A.a.data()));
  return A;
}

// ---- solver.hpp --------------------------------------------------------------
inline CholeskyFactor cholesky(Matrix A, OpCount* ops = nullptr) {
  if (A.rows != A.cols) throw std::invalid_argument("cholesky: matrix not square");
  CholeskyFactor F{Matrix(A.rows, A.cols)};
  int64_t piv = -1;
  const int rc = pkrrgpu_cholesky(default_engine().get(), A.a.data(), A.rows, F.L.a.data(), &piv);
  detail::check(rc, piv);
  if (ops) {
    const std::uint64_t mu = A.rows;
    ops->solve_flops += mu * (mu + 1) * (2 * mu + 1) / 6;
  }
  return F;
}

inline std::vector<double> solve_spd(const CholeskyFactor& F, std::span<const double> b,
                                     OpCount* ops = nullptr) {
  if (b.size() != F.L.rows) throw std::invalid_argument("solve_spd: size mismatch");
  std::vector<double> x(F.L.rows);
  detail::check(pkrrgpu_solve_spd(default_engine().get(), F.L.a.data(), F.L.rows, b.data(), x.data()));
  if (ops) {
    const std::uint64_t mu = F.L.rows;
    ops->solve_flops += 2 * mu * mu;
  }
  return x;
}

inline KrrModel train_krr(const Dataset& data, const KernelSpec& spec, double lambda, OpCount* ops = nullptr) {
  if (data.n == 0) throw std::invalid_argument("train_krr: empty dataset");
  if (!(lambda > 0.0)) throw std::invalid_argument("train_krr: lambda must be > 0");
  detail::require_gaussian(spec);
  const std::vector<double> X = detail::dense(data);
  KrrModel model;
  model.alpha.resize(data.n);
  int64_t piv = -1;
  const int rc = pkrrgpu_train_krr(default_engine().get(), X.data(), data.y.data(), data.n, data.d, spec.sigma,
                                   lambda, model.alpha.data(), &model.residual_ratio, &piv);
  detail::check(rc, piv);
  model.support = data;
  model.support_sq_norms.resize(data.n);
  for (std::size_t i = 0; i < data.n; ++i) model.support_sq_norms[i] = squared_norm(data.row(i));
  model.kernel = spec;
  model.lambda = lambda;
  OpCount local;  // solver.cpp:89-125 charges: gram + shift + factor + solves
  {
    std::uint64_t f = 0;
    for (std::size_t i = 0; i < data.n; ++i) f += 2 * data.row(i).nnz();
    for (std::size_t i = 0; i < data.n; ++i)
      for (std::size_t j = i; j < data.n; ++j) f += detail::gauss_pair_flops(data.row(i).nnz(), data.row(j).nnz());
    local.gram_flops = f;
    const std::uint64_t mu = data.n;
    local.solve_flops = mu + mu * (mu + 1) * (2 * mu + 1) / 6 + 2 * mu * mu;
  }
  model.train_ops = local;
  if (ops) *ops += local;
  return model;
}

// ---- clustering.hpp ----------------------------------------------------------
inline Clustering kmeans(const Dataset& X, int k, std::uint64_t seed, const KMeansParams& params = {},
                         KMeansDiag* diag = nullptr) {
  const std::vector<double> D = detail::dense(X);
  Clustering c;
  c.k = k;
  c.d = X.d;
  c.membership.resize(X.n);
  std::vector<double> centers(static_cast<std::size_t>(k > 0 ? k : 0) * X.d);
  std::vector<int64_t> sizes(k > 0 ? k : 0);
  int iters = 0;
  detail::check(pkrrgpu_kmeans(default_engine().get(), D.data(), X.n, X.d, k, seed, params.threshold,
                               params.max_iters, c.membership.data(), centers.data(), sizes.data(), &iters));
  for (int j = 0; j < k; ++j) {
    c.centers.emplace_back(centers.begin() + j * X.d, centers.begin() + (j + 1) * X.d);
    c.sizes.push_back(static_cast<std::size_t>(sizes[j]));
  }
  if (diag) diag->iterations = iters;  // per-iteration WCSS is not recorded on the GPU path
  return c;
}

inline Clustering kbalance(const Dataset& X, int k, std::uint64_t seed, const KMeansParams& params = {}) {
  const std::vector<double> D = detail::dense(X);
  Clustering c;
  c.k = k;
  c.d = X.d;
  c.membership.resize(X.n);
  std::vector<double> centers(static_cast<std::size_t>(k > 0 ? k : 0) * X.d);
  std::vector<int64_t> sizes(k > 0 ? k : 0);
  detail::check(pkrrgpu_kbalance(default_engine().get(), D.data(), X.n, X.d, k, seed, params.threshold,
                                 params.max_iters, params.recompute_centers ? 1 : 0, c.membership.data(),
                                 centers.data(), sizes.data()));
  for (int j = 0; j < k; ++j) {
    c.centers.emplace_back(centers.begin() + j * X.d, centers.begin() + (j + 1) * X.d);
    c.sizes.push_back(static_cast<std::size_t>(sizes[j]));
  }
  return c;
}

inline int nearest_center(const std::vector<std::vector<double>>& centers, SparseRow x) {
  if (centers.empty()) throw std::invalid_argument("nearest_center: no centers");
  const std::size_t d = centers[0].size();
  std::vector<double> C;
  for (const auto& c : centers) C.insert(C.end(), c.begin(), c.end());
  std::vector<double> q(d, 0.0);
  for (std::size_t k = 0; k < x.nnz(); ++k) q[x.idx[k]] = x.val[k];
  int32_t out = 0;
  detail::check(pkrrgpu_nearest_center(default_engine().get(), C.data(), static_cast<int>(centers.size()), d,
                                       q.data(), 1, &out));
  return out;
}

inline int nearest_center(const Clustering& c, SparseRow x) { return gpu::nearest_center(c.centers, x); }

// ---- dataset.hpp: load_libsvm (dataset.cpp:83-125), host threads -------------------
inline Dataset load_libsvm(const std::string& path) {
  pkrrgpu_dataset* h = nullptr;
  const int rc = pkrrgpu_load_libsvm(path.c_str(), 0, &h);
  if (rc == PKRRGPU_IO) throw std::runtime_error(pkrrgpu_last_error());
  detail::check(rc);
  int64_t n = 0, d = 0, nnz = 0;
  pkrrgpu_dataset_shape(h, &n, &d, &nnz);
  std::vector<int64_t> rp(n + 1);
  Dataset ds;
  ds.col.resize(nnz);
  ds.val.resize(nnz);
  ds.y.resize(n);
  pkrrgpu_dataset_csr(h, rp.data(), ds.col.data(), ds.val.data(), ds.y.data());
  pkrrgpu_dataset_free(h);
  ds.row_ptr.assign(rp.begin(), rp.end());
  ds.n = static_cast<std::size_t>(n);
  ds.d = static_cast<std::size_t>(d);
  return ds;
}

// ---- dataset.hpp: standardize (dataset.cpp:199-232) ---------------------------
inline StandardizeResult standardize(const Dataset& train, const Dataset& test) {
  if (train.n == 0) throw std::invalid_argument("standardize: empty training set");
  if (test.n > 0 && test.d > train.d)
    throw std::invalid_argument("standardize: test dimension exceeds train dimension");
  const std::size_t d = train.d;
  const std::vector<double> X = detail::dense(train);
  std::vector<double> T(test.n * d, 0.0);  // test rows widened to train.d (extra columns dropped below)
  for (std::size_t i = 0; i < test.n; ++i) {
    const SparseRow r = test.row(i);
    for (std::size_t k = 0; k < r.nnz(); ++k) T[i * d + r.idx[k]] = r.val[k];
  }
  std::vector<double> Xo(X.size()), To(T.size());
  StandardizeResult out;
  out.stats.mean.resize(d);
  out.stats.stddev.resize(d);
  detail::check(pkrrgpu_standardize(default_engine().get(), X.data(), train.n, d, test.n ? T.data() : nullptr,
                                    test.n, Xo.data(), test.n ? To.data() : nullptr, out.stats.mean.data(),
                                    out.stats.stddev.data()));
  auto emit = [](Dataset& ds, const std::vector<double>& V, std::size_t rows, std::size_t ld, std::size_t w,
                 const std::vector<double>& y) {  // apply_feature_stats' dense rows (dataset.cpp:183-193)
    ds.d = w;
    std::vector<int> idx(w);
    for (std::size_t j = 0; j < w; ++j) idx[j] = static_cast<int>(j);
    for (std::size_t i = 0; i < rows; ++i) ds.add_row(idx, std::span<const double>(V.data() + i * ld, w), y[i]);
    ds.d = w;
  };
  emit(out.train, Xo, train.n, d, d, train.y);
  if (test.n > 0) {
    emit(out.test, To, test.n, d, test.d, test.y);
    if (test.d < train.d) out.test.d = train.d;  // dataset.cpp:229
  }
  return out;
}

// ---- strategies.hpp ----------------------------------------------------------
inline std::vector<double> auto_sigma_grid(const Dataset& train, std::uint64_t seed) {
  const std::vector<double> X = detail::dense(train);
  std::vector<double> g(9);
  detail::check(pkrrgpu_auto_sigma_grid(default_engine().get(), train.n ? X.data() : nullptr, train.n, train.d,
                                        seed, g.data()));
  return g;
}

inline PartitionSet make_partition(StrategyKind kind, const Dataset& train, std::size_t p, std::uint64_t seed) {
  const std::vector<double> D = detail::dense(train);
  std::vector<int32_t> part_of(train.n);
  std::vector<int64_t> order(train.n);
  std::vector<double> centers((p > 0 ? p : 1) * train.d);
  int64_t pe = 0;
  detail::check(pkrrgpu_make_partition(default_engine().get(), static_cast<int>(kind), D.data(), train.n, train.d,
                                       p, seed, part_of.data(), order.data(), centers.data(), &pe));
  PartitionSet ps;
  ps.p = static_cast<std::size_t>(pe);
  std::vector<std::size_t> sizes(ps.p, 0);
  for (int32_t t : part_of) ++sizes[t];
  std::size_t at = 0;
  for (std::size_t t = 0; t < ps.p; ++t) {
    ps.parts.emplace_back(order.begin() + at, order.begin() + at + sizes[t]);
    at += sizes[t];
  }
  const PartitionerKind pk = partitioner_for(kind);
  if (pk == PartitionerKind::kmeans || pk == PartitionerKind::kbalance)
    for (std::size_t t = 0; t < ps.p; ++t)
      ps.centers.emplace_back(centers.begin() + t * train.d, centers.begin() + (t + 1) * train.d);
  return ps;
}

inline TrainedPartitions train_partitions(const PartitionSet& ps, const Dataset& train, const KernelSpec& spec,
                                          double lambda, std::size_t workers = 1) {
  (void)workers;  // one GPU engine; parts run concurrently on device streams
  for (const auto& part : ps.parts)
    if (part.empty()) throw std::invalid_argument("train_partitions: empty part");
  TrainedPartitions out;
  std::string failures;
  out.stats.per_task.resize(ps.p);
  for (std::size_t t = 0; t < ps.p; ++t) {
    try {
      out.models.push_back(gpu::train_krr(subset(train, ps.parts[t]), spec, lambda, &out.stats.per_task[t].ops));
    } catch (const std::exception& e) {
      out.models.emplace_back();
      if (!failures.empty()) failures += "; ";
      failures += "partition " + std::to_string(t) + ": " + e.what();
    }
  }
  if (!failures.empty()) throw std::runtime_error(failures);
  out.stats.finalize();
  if (ps.has_centers())
    for (std::size_t t = 0; t < ps.p; ++t) out.models[t].center = ps.centers[t];
  return out;
}

// grid_search: the whole per-cell pipeline on the GPU (strategies.cpp:343-507);
// the counters reproduce the reference's accounting (:285-329, :420-452).
inline GridResult grid_search(StrategyKind kind, const Dataset& train, const Dataset& test, std::size_t p,
                              std::span<const double> lambdas, std::span<const double> sigmas, std::uint64_t seed,
                              const GridOptions& options = {}) {
  if (lambdas.empty() || sigmas.empty()) throw std::invalid_argument("grid_search: empty grid");
  if (train.n == 0 || test.n == 0) throw std::invalid_argument("grid_search: empty dataset");
  detail::require_gaussian(options.base_kernel);
  const std::vector<double> Xtr = detail::dense(train), Xte = detail::dense(test);
  const std::size_t nl = lambdas.size(), ns = sigmas.size(), nc = nl * ns;
  const std::size_t pmax = p > 0 ? p : 1;
  std::vector<double> cmse(nc), cres(nc), psse(nc * pmax), pres(nc * pmax);
  std::vector<uint8_t> cfail(nc), pfail(nc * pmax);
  std::vector<int64_t> psizes(pmax), ptest(pmax);
  pkrrgpu_grid_args a{};
  a.strategy = static_cast<int>(kind);
  a.X_train = Xtr.data();
  a.y_train = train.y.data();
  a.n = static_cast<int64_t>(train.n);
  a.d = static_cast<int64_t>(train.d);
  a.X_test = Xte.data();
  a.y_test = test.y.data();
  a.t = static_cast<int64_t>(test.n);
  a.p = static_cast<int64_t>(p);
  a.lambdas = lambdas.data();
  a.n_lambdas = static_cast<int64_t>(nl);
  a.sigmas = sigmas.data();
  a.n_sigmas = static_cast<int64_t>(ns);
  a.seed = seed;
  a.world = 1;
  pkrrgpu_grid_out o{};
  o.cell_mse = cmse.data();
  o.cell_failed = cfail.data();
  o.cell_residual = cres.data();
  o.part_failed = pfail.data();
  o.part_residual = pres.data();
  o.part_sizes = psizes.data();
  o.part_test_count = ptest.data();
  detail::check(pkrrgpu_grid_search_ex(default_engine().get(), &a, &o));
  double ms[8] = {0};
  pkrrgpu_last_timings(default_engine().get(), ms, 8);

  GridResult r;
  r.kind = kind;
  r.p = static_cast<std::size_t>(o.p_effective);
  r.lambdas.assign(lambdas.begin(), lambdas.end());
  r.sigmas.assign(sigmas.begin(), sigmas.end());
  r.cells.resize(nc);
  r.partitions.resize(r.p);
  const PredictorKind predictor = predictor_for(kind);
  const std::uint64_t k_test = test.n, d = train.d;
  for (std::size_t t = 0; t < r.p; ++t) r.partitions[t].size = static_cast<std::size_t>(psizes[t]);
  for (std::size_t si = 0; si < ns; ++si) {
    for (std::size_t li = 0; li < nl; ++li) {
      const std::size_t c = li * ns + si;
      GridCell& cell = r.cells[c];
      cell.lambda = lambdas[li];
      cell.sigma = sigmas[si];
      cell.mse = cmse[c];
      cell.failed = cfail[c] != 0;
      cell.max_residual = cres[c];
      double modeled = 0.0;
      for (std::size_t t = 0; t < r.p; ++t) {
        if (pfail[c * r.p + t] && cell.fail_reason.empty())
          cell.fail_reason = "partition " + std::to_string(t) + ": matrix not positive definite";
        const std::uint64_t m = static_cast<std::uint64_t>(psizes[t]), tt = static_cast<std::uint64_t>(ptest[t]);
        OpCount ops;
        if (!pfail[c * r.p + t]) {  // strategies.cpp:304-329
          ops.solve_flops = m + m * (m + 1) * (2 * m + 1) / 6 + 2 * m * m;
          ops.predict_flops = 2 * tt * m;
        } else {
          ops.solve_flops = m;  // the shift is charged before the factorization throws
        }
        if (li == 0)  // Gram + cross charged to the sigma's first lambda (:285-294, :425)
          ops.gram_flops = 2 * d * m + m * (m + 1) / 2 * (2 * d + 6) + 2 * (m + tt) + tt * m * (2 * d + 6);
        if (r.p > 1) {
          switch (predictor) {
            case PredictorKind::average: ops.messages += 1; ops.bytes += 8 * k_test; break;
            case PredictorKind::nearest: ops.messages += 1; ops.bytes += 8; break;
            case PredictorKind::oracle: ops.messages += k_test; ops.bytes += 8 * k_test; break;
            case PredictorKind::whole: break;
          }
        }
        cell.flops += ops.total_flops();
        cell.messages += ops.messages;
        cell.bytes += ops.bytes;
        const double machine = estimate_time(options.cost, ops);
        if (machine > modeled) modeled = machine;
        PartitionTotals& tot = r.partitions[t];
        tot.ops += ops;
        tot.modeled_seconds += machine;
      }
      cell.modeled_seconds = modeled;
      cell.measured_seconds = ms[3] * 1e-3 / static_cast<double>(nc);  // device time share of the call
    }
  }
  r.best_index = o.best_index < 0 ? GridResult::npos : static_cast<std::size_t>(o.best_index);
  return r;
}

}  // namespace pkrr::gpu
