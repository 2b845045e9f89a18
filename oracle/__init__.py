"""TEST INFRASTRUCTURE ONLY -- parity checkers for the sm_100a path.

Two ctypes front ends with the same Python signatures:

* ``Oracle``    -- oracle/libpkrr_oracle.so, the C restatement (pkrr_oracle.c) of
                   the reference's partitioned Gaussian KRR path.
* ``Reference`` -- oracle/_ref/libpkrr_ref.so, the unmodified reference sources
                   (/root/reference/proj/src) compiled in place + ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg import this package.  The product (paper_1805_00569_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libpkrr_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpkrr_ref.so")

KINDS = {"exact": 0, "dckrr": 1, "kkrr": 2, "kkrr2": 3, "kkrr3": 4, "bkrr": 5, "bkrr2": 6, "bkrr3": 7}

_d = C.POINTER(C.c_double)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)
_u64 = C.POINTER(C.c_uint64)
_u8 = C.POINTER(C.c_uint8)


def build() -> None:
    """Compile the restatement (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _p(a, t):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class NotPositiveDefinite(RuntimeError):
    def __init__(self, pivot):
        super().__init__(f"matrix not positive definite: pivot {pivot}")
        self.pivot = int(pivot)


class _Base:
    prefix = ""

    def _fn(self, name, restype, *argtypes):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        f.argtypes = list(argtypes)
        return f

    # ---- kernel -----------------------------------------------------------
    def gram_sym(self, X, sigma):
        X = _f64(X)
        m, d = X.shape
        K = np.empty((m, m))
        self._gram_sym(_p(X, _d), m, d, float(sigma), _p(K, _d))
        return K

    def gram_cross(self, A, B, sigma):
        A, B = _f64(A), _f64(B)
        K = np.empty((A.shape[0], B.shape[0]))
        self._gram_cross(_p(A, _d), A.shape[0], _p(B, _d), B.shape[0], A.shape[1], float(sigma), _p(K, _d))
        return K

    # ---- clustering -------------------------------------------------------
    def kmeans(self, X, k, seed, threshold=0.01, max_iters=100, want_wcss=False):
        X = _f64(X)
        n, d = X.shape
        mem = np.empty(n, np.int32)
        cen = np.empty((k, d))
        sz = np.empty(k, np.int64)
        it = C.c_int(0)
        wcss = np.zeros(max(max_iters, 1))
        st = self._kmeans(_p(X, _d), n, d, k, seed, threshold, max_iters, _p(mem, _i32), _p(cen, _d),
                          _p(sz, _i64), C.byref(it), _p(wcss, _d) if want_wcss else None)
        if st:
            raise ValueError("kmeans: need 1 <= k <= n")
        out = dict(membership=mem, centers=cen, sizes=sz, iterations=it.value)
        if want_wcss:
            out["wcss"] = wcss[: it.value].copy()
        return out

    def kbalance(self, X, k, seed, threshold=0.01, max_iters=100, recompute=True):
        X = _f64(X)
        n, d = X.shape
        mem = np.empty(n, np.int32)
        cen = np.empty((k, d))
        sz = np.empty(k, np.int64)
        st = self._kbalance(_p(X, _d), n, d, k, seed, threshold, max_iters, int(recompute), _p(mem, _i32),
                            _p(cen, _d), _p(sz, _i64))
        if st:
            raise ValueError(f"kbalance failed ({st})")
        return dict(membership=mem, centers=cen, sizes=sz)

    def nearest_center(self, centers, x):
        centers, x = _f64(centers), _f64(x)
        return int(self._nearest(_p(centers, _d), centers.shape[0], centers.shape[1], _p(x, _d)))

    # ---- data preparation (dataset.cpp:199-232, strategies.cpp:204-234) -----
    def standardize(self, Xtr, Xte=None):
        Xtr = _f64(Xtr)
        n, d = Xtr.shape
        Xte = np.zeros((0, d)) if Xte is None else _f64(Xte)
        tr, te = np.zeros_like(Xtr), np.zeros_like(Xte)
        mean, sd = np.empty(d), np.empty(d)
        st = self._standardize(_p(Xtr, _d), n, d, _p(Xte, _d), Xte.shape[0], _p(tr, _d), _p(te, _d),
                               _p(mean, _d), _p(sd, _d))
        if st:
            raise ValueError("standardize failed")
        return tr, te, mean, sd

    def auto_sigma_grid(self, X, seed):
        X = _f64(X)
        g = np.empty(9)
        self._sigma_grid(_p(X, _d), X.shape[0], X.shape[1], seed, _p(g, _d))
        return g

    def make_partition(self, kind, X, p, seed):
        X = _f64(X)
        n, d = X.shape
        part = np.empty(n, np.int32)
        cen = np.zeros((max(p, 1), d))
        pe = self._make_partition(KINDS[kind], _p(X, _d), n, d, p, seed, _p(part, _i32), _p(cen, _d))
        if pe < 0:
            raise ValueError("make_partition failed")
        return part, cen[:pe]


class Oracle(_Base):
    """C restatement of the reference path (pkrr_oracle.c)."""

    prefix = "pko_"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        self._gram_sym = self._fn("gram_sym", None, _d, C.c_int64, C.c_int64, C.c_double, _d)
        self._gram_cross = self._fn("gram_cross", None, _d, C.c_int64, _d, C.c_int64, C.c_int64, C.c_double, _d)
        self._chol = self._fn("cholesky", C.c_int, _d, C.c_int64, _i64, _d)
        self._solve = self._fn("solve_spd", None, _d, C.c_int64, _d, _d)
        self._train = self._fn("train_krr", C.c_int, _d, _d, C.c_int64, C.c_int64, C.c_double, C.c_double,
                               _d, _d, _i64)
        self._predict = self._fn("predict", C.c_double, _d, _d, _d, C.c_int64, C.c_int64, C.c_double, _d)
        self._kmeans = self._fn("kmeans", C.c_int, _d, C.c_int64, C.c_int64, C.c_int, C.c_uint64, C.c_double,
                                C.c_int, _i32, _d, _i64, C.POINTER(C.c_int), _d)
        self._kbalance = self._fn("kbalance", C.c_int, _d, C.c_int64, C.c_int64, C.c_int, C.c_uint64,
                                  C.c_double, C.c_int, C.c_int, _i32, _d, _i64)
        self._nearest = self._fn("nearest_center", C.c_int, _d, C.c_int, C.c_int64, _d)
        self._make_partition = self._fn("make_partition", C.c_int64, C.c_int, _d, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_uint64, _i32, _i64, _d)
        self._grid = self._fn("grid_search", C.c_int64, C.c_int, _d, _d, C.c_int64, C.c_int64, _d, _d,
                              C.c_int64, C.c_int64, _d, C.c_int64, _d, C.c_int64, C.c_uint64, _d, _u8, _d,
                              _i32, _d, _d)
        self._grid_parts = self._fn("grid_search_parts", C.c_int64, C.c_int, _d, _d, C.c_int64, C.c_int64,
                                    _d, _d, C.c_int64, C.c_int64, _i32, _i64, _d, _d, C.c_int64, _d,
                                    C.c_int64, _d, _u8, _d, _d)
        self._mse = self._fn("mse", C.c_double, _d, _d, C.c_int64)
        self._sub_seed = self._fn("sub_seed", C.c_uint64, C.c_uint64, C.c_char_p)
        self._sqnorm = self._fn("squared_norm", C.c_double, _d, C.c_int64)
        self._resid = self._fn("residual_slice", C.c_double, _d, C.c_int64, C.c_double, _d, _d)
        _std = self._fn("standardize", None, _d, C.c_int64, C.c_int64, _d, C.c_int64, _d, _d, _d, _d)
        self._standardize = lambda *a: (_std(*a), 0)[1]
        self._sigma_grid = self._fn("auto_sigma_grid", None, _d, C.c_int64, C.c_int64, C.c_uint64, _d)

    def cholesky(self, A):
        L = _f64(A).copy()
        piv = C.c_int64(-1)
        if self._chol(_p(L, _d), L.shape[0], C.byref(piv), None):
            raise NotPositiveDefinite(piv.value)
        return L

    def solve_spd(self, L, b):
        L, b = _f64(L), _f64(b)
        x = np.empty(L.shape[0])
        self._solve(_p(L, _d), L.shape[0], _p(b, _d), _p(x, _d))
        return x

    def train_krr(self, X, y, sigma, lam):
        X, y = _f64(X), _f64(y)
        m, d = X.shape
        alpha = np.empty(m)
        res = C.c_double(0)
        piv = C.c_int64(-1)
        st = self._train(_p(X, _d), _p(y, _d), m, d, sigma, lam, _p(alpha, _d), C.byref(res), C.byref(piv))
        if st == 2:
            raise NotPositiveDefinite(piv.value)
        if st:
            raise ValueError("train_krr: invalid argument")
        return alpha, res.value

    def predict(self, S, alpha, sigma, Q):
        S, alpha, Q = _f64(S), _f64(alpha), _f64(Q)
        m, d = S.shape
        sn = np.array([self._sqnorm(_p(np.ascontiguousarray(S[i]), _d), d) for i in range(m)])
        out = np.empty(Q.shape[0])
        for j in range(Q.shape[0]):
            q = np.ascontiguousarray(Q[j])
            out[j] = self._predict(_p(S, _d), _p(sn, _d), _p(alpha, _d), m, d, sigma, _p(q, _d))
        return out

    def residual_slice(self, K, shift, alpha, y):
        K, alpha, y = _f64(K), _f64(alpha), _f64(y)
        return float(self._resid(_p(K, _d), K.shape[0], shift, _p(alpha, _d), _p(y, _d)))

    def mse(self, pred, truth):
        pred, truth = _f64(pred), _f64(truth)
        return float(self._mse(_p(pred, _d), _p(truth, _d), pred.shape[0]))

    def sub_seed(self, seed, tag):
        return int(self._sub_seed(seed, tag.encode()))

    def grid_search(self, kind, Xtr, ytr, Xte, yte, p, lambdas, sigmas, seed):
        Xtr, ytr, Xte, yte = _f64(Xtr), _f64(ytr), _f64(Xte), _f64(yte)
        lam, sig = _f64(lambdas), _f64(sigmas)
        n, d = Xtr.shape
        t = Xte.shape[0]
        nc = lam.size * sig.size
        mse = np.empty(nc)
        failed = np.zeros(nc, np.uint8)
        res = np.zeros(nc)
        part = np.empty(n, np.int32)
        cen = np.zeros((max(p, 1), d))
        best_pred = np.zeros(t)
        best = self._grid(KINDS[kind], _p(Xtr, _d), _p(ytr, _d), n, d, _p(Xte, _d), _p(yte, _d), t, p,
                          _p(lam, _d), lam.size, _p(sig, _d), sig.size, seed, _p(mse, _d), _p(failed, _u8),
                          _p(res, _d), _p(part, _i32), _p(cen, _d), _p(best_pred, _d))
        return dict(best=int(best), mse=mse, failed=failed.astype(bool), residual=res, part_of=part,
                    centers=cen, best_pred=best_pred)

    # ---- data preparation (dataset.cpp:199-232, strategies.cpp:204-234) -----
    def standardize(self, Xtr, Xte=None):
        Xtr = _f64(Xtr)
        n, d = Xtr.shape
        Xte = np.zeros((0, d)) if Xte is None else _f64(Xte)
        tr, te = np.zeros_like(Xtr), np.zeros_like(Xte)
        mean, sd = np.empty(d), np.empty(d)
        st = self._standardize(_p(Xtr, _d), n, d, _p(Xte, _d), Xte.shape[0], _p(tr, _d), _p(te, _d),
                               _p(mean, _d), _p(sd, _d))
        if st:
            raise ValueError("standardize failed")
        return tr, te, mean, sd

    def auto_sigma_grid(self, X, seed):
        X = _f64(X)
        g = np.empty(9)
        self._sigma_grid(_p(X, _d), X.shape[0], X.shape[1], seed, _p(g, _d))
        return g

    def make_partition(self, kind, X, p, seed):
        """Returns (part_of, order, centers); order = rows part by part."""
        X = _f64(X)
        n, d = X.shape
        part = np.empty(n, np.int32)
        order = np.empty(n, np.int64)
        cen = np.zeros((max(p, 1), d))
        pe = self._make_partition(KINDS[kind], _p(X, _d), n, d, p, seed, _p(part, _i32), _p(order, _i64),
                                  _p(cen, _d))
        if pe < 0:
            raise ValueError("make_partition failed")
        return part, order, cen[:pe]

    def grid_search_parts(self, kind, Xtr, ytr, Xte, yte, part_of, centers, lambdas, sigmas, order=None):
        Xtr, ytr, Xte, yte = _f64(Xtr), _f64(ytr), _f64(Xte), _f64(yte)
        lam, sig = _f64(lambdas), _f64(sigmas)
        part_of = np.ascontiguousarray(part_of, np.int32)
        if order is None:
            order = np.argsort(part_of, kind="stable")
        order = np.ascontiguousarray(order, np.int64)
        centers = _f64(centers)
        n, d = Xtr.shape
        t = Xte.shape[0]
        p = int(part_of.max()) + 1
        nc = lam.size * sig.size
        mse = np.empty(nc)
        failed = np.zeros(nc, np.uint8)
        res = np.zeros(nc)
        best_pred = np.zeros(t)
        best = self._grid_parts(KINDS[kind], _p(Xtr, _d), _p(ytr, _d), n, d, _p(Xte, _d), _p(yte, _d), t, p,
                                _p(part_of, _i32), _p(order, _i64), _p(centers, _d), _p(lam, _d), lam.size,
                                _p(sig, _d), sig.size,
                                _p(mse, _d), _p(failed, _u8), _p(res, _d), _p(best_pred, _d))
        return dict(best=int(best), mse=mse, failed=failed.astype(bool), residual=res, best_pred=best_pred)


class Reference(_Base):
    """The unmodified reference library (oracle/_ref/libpkrr_ref.so)."""

    prefix = "ref_"

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_SO):
        self.lib = C.CDLL(path)
        self._gram_sym = self._fn("gram_sym", C.c_int, _d, C.c_int64, C.c_int64, C.c_double, _d)
        self._gram_cross = self._fn("gram_cross", C.c_int, _d, C.c_int64, _d, C.c_int64, C.c_int64, C.c_double, _d)
        self._chol = self._fn("cholesky", C.c_int, _d, C.c_int64, _d, _i64)
        self._solve = self._fn("solve_spd", None, _d, C.c_int64, _d, _d)
        self._train = self._fn("train_krr", C.c_int, _d, _d, C.c_int64, C.c_int64, C.c_double, C.c_double,
                               _d, _d, _i64)
        self._train_predict = self._fn("train_predict", C.c_int, _d, _d, C.c_int64, C.c_int64, C.c_double,
                                       C.c_double, _d, C.c_int64, _d)
        self._kmeans = self._fn("kmeans", C.c_int, _d, C.c_int64, C.c_int64, C.c_int, C.c_uint64, C.c_double,
                                C.c_int, _i32, _d, _i64, C.POINTER(C.c_int), _d)
        self._kbalance = self._fn("kbalance", C.c_int, _d, C.c_int64, C.c_int64, C.c_int, C.c_uint64,
                                  C.c_double, C.c_int, C.c_int, _i32, _d, _i64)
        self._nearest = self._fn("nearest_center", C.c_int, _d, C.c_int, C.c_int64, _d)
        self._make_partition = self._fn("make_partition", C.c_int64, C.c_int, _d, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_uint64, _i32, _d)
        self._grid = self._fn("grid_search", C.c_int64, C.c_int, _d, _d, C.c_int64, C.c_int64, _d, _d,
                              C.c_int64, C.c_int64, _d, C.c_int64, _d, C.c_int64, C.c_uint64, C.c_int64, _d,
                              _u8, _d)
        self._tpn = self._fn("train_predict_nearest", C.c_int, C.c_int, _d, _d, C.c_int64, C.c_int64,
                             C.c_int64, C.c_uint64, C.c_double, C.c_double, C.c_int64, _d, C.c_int64, _d)
        self._sub_seed = self._fn("sub_seed", C.c_uint64, C.c_uint64, C.c_char_p)
        self._stream = self._fn("rng_stream", None, C.c_uint64, C.c_int64, _d, _u64, C.c_uint64)
        self._perm = self._fn("random_permutation", None, C.c_uint64, C.c_int64, _u64)
        self._err = self._fn("last_error", C.c_char_p)
        self._standardize = self._fn("standardize", C.c_int, _d, C.c_int64, C.c_int64, _d, C.c_int64, _d, _d,
                                     _d, _d)
        self._sigma_grid = self._fn("auto_sigma_grid", C.c_int, _d, C.c_int64, C.c_int64, C.c_uint64, _d)
        self._libsvm = self._fn("load_libsvm", C.c_int, C.c_char_p, _i64, _i64, _i64, _i64, _i32, _d, _d)
        self._tpp = self._fn("train_partitions_predict", C.c_int, _d, _d, C.c_int64, C.c_int64, _i32, C.c_int64,
                             _d, C.c_double, C.c_double, C.c_int64, _d, C.c_int64, _d, _d, _d, _d)

    def train_partitions_predict(self, Xtr, ytr, part_of, p, centers, sigma, lam, Q, workers=1):
        """strategies.cpp:104-149 with a caller-given partition: train_partitions(ps, ...)
        then predict_nearest (centers given) / the single model.  Returns (alpha
        concatenated part by part, residual[p], predictions[q], task seconds[p])."""
        Xtr, ytr, Q = _f64(Xtr), _f64(ytr), _f64(Q)
        part_of = np.ascontiguousarray(part_of, np.int32)
        n, d = Xtr.shape
        cen = None if centers is None else _f64(centers)
        alpha, res, sec = np.empty(n), np.empty(p), np.empty(p)
        pred = np.empty(Q.shape[0])
        st = self._tpp(_p(Xtr, _d), _p(ytr, _d), n, d, _p(part_of, _i32), p, None if cen is None else _p(cen, _d),
                       sigma, lam, workers, _p(Q, _d), Q.shape[0], _p(alpha, _d), _p(res, _d), _p(pred, _d),
                       _p(sec, _d))
        if st == 2:
            raise NotPositiveDefinite(-1)
        if st:
            raise RuntimeError(self._err().decode())
        return alpha, res, pred, sec

    def load_libsvm(self, path):
        """dataset.cpp:83-125: (row_ptr, col, val, y, d) exactly as the reference's Dataset."""
        n, d, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        if self._libsvm(path.encode(), C.byref(n), C.byref(d), C.byref(nnz), None, None, None, None):
            raise RuntimeError(self._err().decode())
        rp, col = np.empty(n.value + 1, np.int64), np.empty(nnz.value, np.int32)
        val, y = np.empty(nnz.value), np.empty(n.value)
        self._libsvm(path.encode(), C.byref(n), C.byref(d), C.byref(nnz), _p(rp, _i64), _p(col, _i32), _p(val, _d),
                     _p(y, _d))
        return rp, col, val, y, d.value

    def cholesky(self, A):
        A = _f64(A)
        L = np.empty_like(A)
        piv = C.c_int64(-1)
        st = self._chol(_p(A, _d), A.shape[0], _p(L, _d), C.byref(piv))
        if st == 2:
            raise NotPositiveDefinite(piv.value)
        return L

    def solve_spd(self, L, b):
        L, b = _f64(L), _f64(b)
        x = np.empty(L.shape[0])
        self._solve(_p(L, _d), L.shape[0], _p(b, _d), _p(x, _d))
        return x

    def train_krr(self, X, y, sigma, lam):
        X, y = _f64(X), _f64(y)
        m, d = X.shape
        alpha = np.empty(m)
        res = C.c_double(0)
        piv = C.c_int64(-1)
        st = self._train(_p(X, _d), _p(y, _d), m, d, sigma, lam, _p(alpha, _d), C.byref(res), C.byref(piv))
        if st == 2:
            raise NotPositiveDefinite(piv.value)
        if st:
            raise ValueError(self._err().decode())
        return alpha, res.value

    def train_predict(self, X, y, sigma, lam, Q):
        X, y, Q = _f64(X), _f64(y), _f64(Q)
        out = np.empty(Q.shape[0])
        if self._train_predict(_p(X, _d), _p(y, _d), X.shape[0], X.shape[1], sigma, lam, _p(Q, _d), Q.shape[0],
                               _p(out, _d)):
            raise RuntimeError(self._err().decode())
        return out

    def train_predict_nearest(self, kind, Xtr, ytr, p, seed, sigma, lam, Q, workers=1):
        Xtr, ytr, Q = _f64(Xtr), _f64(ytr), _f64(Q)
        out = np.empty(Q.shape[0])
        if self._tpn(KINDS[kind], _p(Xtr, _d), _p(ytr, _d), Xtr.shape[0], Xtr.shape[1], p, seed, sigma, lam,
                     workers, _p(Q, _d), Q.shape[0], _p(out, _d)):
            raise RuntimeError(self._err().decode())
        return out

    def grid_search(self, kind, Xtr, ytr, Xte, yte, p, lambdas, sigmas, seed, workers=1):
        Xtr, ytr, Xte, yte = _f64(Xtr), _f64(ytr), _f64(Xte), _f64(yte)
        lam, sig = _f64(lambdas), _f64(sigmas)
        nc = lam.size * sig.size
        mse = np.empty(nc)
        failed = np.zeros(nc, np.uint8)
        res = np.zeros(nc)
        best = self._grid(KINDS[kind], _p(Xtr, _d), _p(ytr, _d), Xtr.shape[0], Xtr.shape[1], _p(Xte, _d),
                          _p(yte, _d), Xte.shape[0], p, _p(lam, _d), lam.size, _p(sig, _d), sig.size, seed,
                          workers, _p(mse, _d), _p(failed, _u8), _p(res, _d))
        if best == -2:
            raise RuntimeError(self._err().decode())
        return dict(best=int(best), mse=mse, failed=failed.astype(bool), residual=res)

    def sub_seed(self, seed, tag):
        return int(self._sub_seed(seed, tag.encode()))

    def rng_stream(self, seed, count, below_n):
        normals = np.empty(count)
        belows = np.empty(count, np.uint64)
        self._stream(seed, count, _p(normals, _d), _p(belows, _u64), below_n)
        return normals, belows

    def random_permutation(self, seed, n):
        perm = np.empty(n, np.uint64)
        self._perm(seed, n, _p(perm, _u64))
        return perm
