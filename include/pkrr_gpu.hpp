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
//   double        predict_nearest(models, centers, x, ops)  strategies.hpp:56-58
//   double        predict_average(models, x, ops)           :54-55
//   pair          predict_oracle(models, x, y_true, ops)    :59-62
//   GridResult    grid_search(kind, train, test, p, lambdas, sigmas, seed, options)  :117-120
//
// Batched GPU-resident forms of the predict stage: DeviceModels (train_partitions_device)
// with predict_nearest(DeviceModels, Q) / predict(DeviceModels, t, Q), and
// predict_nearest(models, centers, const Dataset& Q) over host KrrModels.
//
// Devices: every call runs on default_group() -- one engine context per GPU (env
// PKRR_GPUS = a count "4" or a device list "0,1,2,3"; default: every visible GPU) with
// one host thread per GPU.  grid_search shards the parts over the group's GPUs (bitwise
// the one-GPU result), so the reference's multi-worker callers (cmd_run, cmd_weak_scaling,
// experiment.cpp:107-110,272-274) scale over the GPUs unchanged.  Single-matrix calls use
// the group's first GPU.
// The analytic OpCount charges follow the reference accounting exactly
// (kernel.cpp:68-79, solver.cpp:39-42/67-70, strategies.cpp:285-329/420-452), so
// counters, messages, bytes and modeled_seconds in GridResult are identical.
// Requires the reference headers on the include path and libpkrr_gpu.so at link.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <limits>
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

// ---- engine handles ----------------------------------------------------------
// One context per GPU, one host thread per GPU inside the library (pkrrgpu_multi).
class Group {
 public:
  explicit Group(const std::vector<int>& devices) {
    if (pkrrgpu_multi_create(devices.data(), static_cast<int>(devices.size()), &m_) != PKRRGPU_OK)
      throw std::runtime_error(std::string("pkrr-gpu: ") + pkrrgpu_last_error());
  }
  ~Group() { pkrrgpu_multi_destroy(m_); }
  Group(const Group&) = delete;
  Group& operator=(const Group&) = delete;
  pkrrgpu_multi* get() const { return m_; }
  int size() const { return pkrrgpu_multi_size(m_); }
  pkrrgpu_ctx* context(int i = 0) const { return pkrrgpu_multi_context(m_, i); }

 private:
  pkrrgpu_multi* m_ = nullptr;
};

namespace detail {
inline std::vector<int> default_devices() {
  std::vector<int> devs;
  if (const char* e = std::getenv("PKRR_GPUS")) {
    const std::string s(e);
    if (s.find(',') == std::string::npos) {
      const int n = std::atoi(s.c_str());
      for (int i = 0; i < n; ++i) devs.push_back(i);
    } else {
      std::size_t at = 0;
      while (at <= s.size()) {
        const std::size_t c = s.find(',', at);
        devs.push_back(std::atoi(s.substr(at, c == std::string::npos ? std::string::npos : c - at).c_str()));
        if (c == std::string::npos) break;
        at = c + 1;
      }
    }
  }
  if (devs.empty()) {
    const int n = pkrrgpu_device_count();
    for (int i = 0; i < (n > 0 ? n : 1); ++i) devs.push_back(i);
  }
  return devs;
}
}  // namespace detail

inline Group& default_group() {
  static Group g(detail::default_devices());
  return g;
}

// the group's first context (single-matrix primitives)
struct EngineRef {
  pkrrgpu_ctx* ctx;
  pkrrgpu_ctx* get() const { return ctx; }
};
inline EngineRef default_engine() { return EngineRef{default_group().context(0)}; }

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

namespace detail {
// OpCount charges of train_krr (solver.cpp:89-125): gram + shift + factor + solves
inline OpCount train_ops(const Dataset& data) {
  OpCount local;
  std::uint64_t f = 0;
  for (std::size_t i = 0; i < data.n; ++i) f += 2 * data.row(i).nnz();
  for (std::size_t i = 0; i < data.n; ++i)
    for (std::size_t j = i; j < data.n; ++j) f += gauss_pair_flops(data.row(i).nnz(), data.row(j).nnz());
  local.gram_flops = f;
  const std::uint64_t mu = data.n;
  local.solve_flops = mu + mu * (mu + 1) * (2 * mu + 1) / 6 + 2 * mu * mu;
  return local;
}

// KrrModel::predict charges for one row (solver.cpp:74-87)
inline std::uint64_t predict_row_flops(const KrrModel& m, SparseRow x) {
  std::uint64_t f = 2 * x.nnz();
  for (std::size_t i = 0; i < m.support.n; ++i) f += gauss_pair_flops(m.support.row(i).nnz(), x.nnz()) + 2;
  return f;
}

// ps.parts concatenated + their sizes (the C ABI's PartitionSet)
inline void part_lists(const PartitionSet& ps, std::vector<int64_t>& rows, std::vector<int64_t>& sizes) {
  for (const auto& part : ps.parts) {
    sizes.push_back(static_cast<int64_t>(part.size()));
    for (std::size_t i : part) rows.push_back(static_cast<int64_t>(i));
  }
}

inline std::vector<double> flat_centers(const std::vector<std::vector<double>>& centers) {
  std::vector<double> C;
  for (const auto& c : centers) C.insert(C.end(), c.begin(), c.end());
  return C;
}
}  // namespace detail

// GPU-resident TrainedPartitions: support rows, norms and alpha stay in HBM for the
// batched predict stage (pkrrgpu_models).
class DeviceModels {
 public:
  DeviceModels(pkrrgpu_ctx* ctx, pkrrgpu_models* h, std::size_t d) : ctx_(ctx), h_(h), d_(d) {}
  ~DeviceModels() { pkrrgpu_models_free(h_); }
  DeviceModels(const DeviceModels&) = delete;
  DeviceModels& operator=(const DeviceModels&) = delete;
  DeviceModels(DeviceModels&& o) noexcept : ctx_(o.ctx_), h_(o.h_), d_(o.d_) { o.h_ = nullptr; }
  pkrrgpu_models* get() const { return h_; }
  pkrrgpu_ctx* context() const { return ctx_; }
  std::size_t d() const { return d_; }
  std::size_t size() const { return static_cast<std::size_t>(pkrrgpu_models_count(h_)); }
  std::vector<double> alpha(std::size_t t) const {
    std::vector<double> a(static_cast<std::size_t>(pkrrgpu_models_size(h_, static_cast<int64_t>(t))));
    detail::check(pkrrgpu_models_alpha(h_, static_cast<int64_t>(t), a.data()));
    return a;
  }
  double residual(std::size_t t) const {
    double r = 0.0;
    detail::check(pkrrgpu_models_residual(h_, static_cast<int64_t>(t), &r));
    return r;
  }

 private:
  pkrrgpu_ctx* ctx_;
  pkrrgpu_models* h_;
  std::size_t d_;
};

// train_partitions with the caller's PartitionSet, every part concurrently on the GPU
// (strategies.cpp:104-133); the models stay on the device.
inline DeviceModels train_partitions_device(const PartitionSet& ps, const Dataset& train, const KernelSpec& spec,
                                            double lambda) {
  detail::require_gaussian(spec);
  if (!(lambda > 0.0)) throw std::invalid_argument("train_krr: lambda must be > 0");
  for (const auto& part : ps.parts)
    if (part.empty()) throw std::invalid_argument("train_partitions: empty part");
  const std::vector<double> X = detail::dense(train);
  std::vector<int64_t> rows, sizes;
  detail::part_lists(ps, rows, sizes);
  const std::vector<double> C = detail::flat_centers(ps.centers);
  pkrrgpu_models* h = nullptr;
  int64_t failed = -1, piv = -1;
  pkrrgpu_ctx* ctx = default_engine().get();
  const int rc = pkrrgpu_train_parts(ctx, X.data(), train.y.data(), train.n, train.d, rows.data(), sizes.data(),
                                     ps.p, ps.has_centers() ? C.data() : nullptr, spec.sigma, lambda, &h, &failed,
                                     &piv);
  if (rc == PKRRGPU_NPD)  // train_partitions aggregates solver failures by part (strategies.cpp:119-125)
    throw std::runtime_error("partition " + std::to_string(failed) + ": " + pkrrgpu_last_error());
  detail::check(rc, piv);
  return DeviceModels(ctx, h, train.d);
}

inline TrainedPartitions train_partitions(const PartitionSet& ps, const Dataset& train, const KernelSpec& spec,
                                          double lambda, std::size_t workers = 1) {
  (void)workers;  // every part runs concurrently on the device's streams
  const DeviceModels dm = train_partitions_device(ps, train, spec, lambda);
  TrainedPartitions out;
  out.stats.per_task.resize(ps.p);
  for (std::size_t t = 0; t < ps.p; ++t) {
    KrrModel model;
    model.support = subset(train, ps.parts[t]);
    model.support_sq_norms.resize(model.support.n);
    for (std::size_t i = 0; i < model.support.n; ++i) model.support_sq_norms[i] = squared_norm(model.support.row(i));
    model.alpha = dm.alpha(t);
    model.residual_ratio = dm.residual(t);
    model.kernel = spec;
    model.lambda = lambda;
    model.train_ops = detail::train_ops(model.support);
    out.stats.per_task[t].ops = model.train_ops;
    if (ps.has_centers()) model.center = ps.centers[t];
    out.models.push_back(std::move(model));
  }
  out.stats.finalize();
  return out;
}

// ---- predict stage (strategies.hpp:54-62, solver.hpp:48), batched on the GPU --------
namespace detail {
inline std::vector<double> dense_rows(const Dataset& Q, std::size_t d) {
  std::vector<double> X(Q.n * d, 0.0);
  for (std::size_t i = 0; i < Q.n; ++i) {
    const SparseRow r = Q.row(i);
    for (std::size_t k = 0; k < r.nnz(); ++k)
      if (static_cast<std::size_t>(r.idx[k]) < d) X[i * d + r.idx[k]] = r.val[k];
  }
  return X;
}

// host KrrModels -> device models (support rows, alpha, centers)
inline DeviceModels import_models(std::span<const KrrModel> models, const std::vector<std::vector<double>>* centers) {
  if (models.empty()) throw std::invalid_argument("predict: no models");
  const std::size_t d = models[0].support.d;
  std::vector<int64_t> sizes;
  std::vector<double> S, A;
  double sigma = models[0].kernel.sigma;
  for (const KrrModel& m : models) {
    require_gaussian(m.kernel);
    if (m.kernel.sigma != sigma) throw std::invalid_argument("pkrr-gpu: models with different kernels");
    sizes.push_back(static_cast<int64_t>(m.support.n));
    const std::vector<double> X = dense_rows(m.support, d);
    S.insert(S.end(), X.begin(), X.end());
    A.insert(A.end(), m.alpha.begin(), m.alpha.end());
  }
  const std::vector<double> C = centers ? flat_centers(*centers) : std::vector<double>{};
  pkrrgpu_models* h = nullptr;
  pkrrgpu_ctx* ctx = default_engine().get();
  check(pkrrgpu_models_import(ctx, static_cast<int64_t>(models.size()), d, sizes.data(), S.data(), A.data(),
                              centers ? C.data() : nullptr, sigma, &h));
  return DeviceModels(ctx, h, d);
}
}  // namespace detail

// nearest-centre routed predictions of every row of Q over GPU-resident models
inline std::vector<double> predict_nearest(const DeviceModels& models, const Dataset& Q) {
  std::vector<double> out(Q.n);
  if (Q.n == 0) return out;
  const std::vector<double> X = detail::dense_rows(Q, models.d());
  detail::check(pkrrgpu_predict_nearest(models.context(), models.get(), X.data(), Q.n, out.data()));
  return out;
}

// KrrModel::predict of model t over every row of Q
inline std::vector<double> predict(const DeviceModels& models, std::size_t t, const Dataset& Q) {
  std::vector<double> out(Q.n);
  if (Q.n == 0) return out;
  const std::vector<double> X = detail::dense_rows(Q, models.d());
  detail::check(pkrrgpu_models_predict(models.context(), models.get(), static_cast<int64_t>(t), X.data(), Q.n,
                                       out.data()));
  return out;
}

// predict_nearest (strategies.cpp:142-149) over host models, every row of Q at once;
// OpCount charged as the reference's per-row calls would
inline std::vector<double> predict_nearest(std::span<const KrrModel> models,
                                           const std::vector<std::vector<double>>& centers, const Dataset& Q,
                                           OpCount* ops = nullptr) {
  if (models.empty()) throw std::invalid_argument("predict_nearest: no models");
  if (centers.size() != models.size())
    throw std::invalid_argument("predict_nearest: centers undefined for this partitioning");
  const DeviceModels dm = detail::import_models(models, &centers);
  std::vector<double> out = predict_nearest(dm, Q);
  if (ops) {
    const std::vector<double> C = detail::flat_centers(centers), X = detail::dense_rows(Q, dm.d());
    std::vector<int32_t> route(Q.n);
    detail::check(pkrrgpu_nearest_center(dm.context(), C.data(), static_cast<int>(centers.size()), dm.d(), X.data(),
                                         Q.n, route.data()));
    for (std::size_t j = 0; j < Q.n; ++j) ops->predict_flops += detail::predict_row_flops(models[route[j]], Q.row(j));
  }
  return out;
}

// drop-in single-row form (strategies.hpp:56-58)
inline double predict_nearest(std::span<const KrrModel> models, const std::vector<std::vector<double>>& centers,
                              SparseRow x, OpCount* ops = nullptr) {
  Dataset q;
  q.d = models.empty() ? 0 : models[0].support.d;
  q.add_row(std::vector<int>(x.idx.begin(), x.idx.end()), std::span<const double>(x.val.data(), x.val.size()), 0.0);
  q.d = models.empty() ? 0 : models[0].support.d;
  return predict_nearest(models, centers, q, ops)[0];
}

// predict_average (strategies.cpp:135-140): the models' predictions summed in model order / p
inline std::vector<double> predict_average(std::span<const KrrModel> models, const Dataset& Q, OpCount* ops = nullptr) {
  if (models.empty()) throw std::invalid_argument("predict_average: no models");
  const DeviceModels dm = detail::import_models(models, nullptr);
  const std::vector<double> X = detail::dense_rows(Q, dm.d());
  std::vector<double> pp(models.size() * Q.n);
  if (Q.n) detail::check(pkrrgpu_models_predict(dm.context(), dm.get(), -1, X.data(), Q.n, pp.data()));
  std::vector<double> out(Q.n);
  for (std::size_t j = 0; j < Q.n; ++j) {
    double sum = 0.0;
    for (std::size_t t = 0; t < models.size(); ++t) {
      sum += pp[t * Q.n + j];
      if (ops) ops->predict_flops += detail::predict_row_flops(models[t], Q.row(j));
    }
    out[j] = sum / static_cast<double>(models.size());
  }
  return out;
}

inline double predict_average(std::span<const KrrModel> models, SparseRow x, OpCount* ops = nullptr) {
  Dataset q;
  q.d = models.empty() ? 0 : models[0].support.d;
  q.add_row(std::vector<int>(x.idx.begin(), x.idx.end()), std::span<const double>(x.val.data(), x.val.size()), 0.0);
  q.d = models.empty() ? 0 : models[0].support.d;
  return predict_average(models, q, ops)[0];
}

// predict_oracle (strategies.cpp:151-166): the least-squared-error model per row
inline std::vector<std::pair<double, std::size_t>> predict_oracle(std::span<const KrrModel> models, const Dataset& Q,
                                                                  OpCount* ops = nullptr) {
  if (models.empty()) throw std::invalid_argument("predict_oracle: no models");
  const DeviceModels dm = detail::import_models(models, nullptr);
  const std::vector<double> X = detail::dense_rows(Q, dm.d());
  std::vector<double> pp(models.size() * Q.n);
  if (Q.n) detail::check(pkrrgpu_models_predict(dm.context(), dm.get(), -1, X.data(), Q.n, pp.data()));
  std::vector<std::pair<double, std::size_t>> out(Q.n);
  for (std::size_t j = 0; j < Q.n; ++j) {
    double best_pred = 0.0, best_err = std::numeric_limits<double>::infinity();
    std::size_t best_t = 0;
    for (std::size_t t = 0; t < models.size(); ++t) {
      const double pred = pp[t * Q.n + j];
      const double err = (pred - Q.y[j]) * (pred - Q.y[j]);
      if (ops) ops->predict_flops += detail::predict_row_flops(models[t], Q.row(j));
      if (err < best_err) {
        best_err = err;
        best_pred = pred;
        best_t = t;
      }
    }
    out[j] = {best_pred, best_t};
  }
  return out;
}

// grid_search: the whole per-cell pipeline on the GPU (strategies.cpp:343-507);
// the counters reproduce the reference's accounting (:285-329, :420-452).
inline GridResult grid_search(StrategyKind kind, const Dataset& train, const Dataset& test, std::size_t p,
                              std::span<const double> lambdas, std::span<const double> sigmas, std::uint64_t seed,
                              const GridOptions& options = {}, Group& group = default_group()) {
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
  a.world = 1;  // the group shards the parts over its GPUs itself
  pkrrgpu_grid_out o{};
  o.cell_mse = cmse.data();
  o.cell_failed = cfail.data();
  o.cell_residual = cres.data();
  o.part_failed = pfail.data();
  o.part_residual = pres.data();
  o.part_sizes = psizes.data();
  o.part_test_count = ptest.data();
  detail::check(pkrrgpu_multi_grid_search(group.get(), &a, &o));
  double ms[8] = {0};
  for (int g = 0; g < group.size(); ++g) {  // device time: the slowest GPU's
    double mg[8] = {0};
    pkrrgpu_last_timings(group.context(g), mg, 8);
    if (mg[3] > ms[3]) std::copy(mg, mg + 8, ms);
  }

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
