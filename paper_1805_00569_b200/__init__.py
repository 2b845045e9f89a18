"""paper_1805_00569_b200 -- B200 (sm_100a) engine for partitioned Gaussian KRR.

Python mirror of the reference library's hot-path API (arxiv 1805.00569
reference, proj/include/pkrr/*.hpp) over the C ABI in include/pkrr_gpu.h.
Names, argument meaning and error behaviour follow the reference:

    gram(X, Y, sigma)                      kernel.hpp:40  (X is Y -> symmetric path)
    assemble_system(K, lam, m)             kernel.hpp:44
    cholesky(A) -> L                       solver.hpp:29  (raises NotPositiveDefinite)
    solve_spd(L, b)                        solver.hpp:32
    train_krr(X, y, sigma, lam) -> KrrModel solver.hpp:52
    kmeans / kbalance / nearest_center     clustering.hpp:33-45
    make_partition                         strategies.hpp:40
    train_partitions / predict_nearest     strategies.hpp:50-58
    mse                                    strategies.hpp:64
    grid_search -> GridResult              strategies.hpp:117

Every call runs on the GPU through libpkrr_gpu.so; there is no CPU fallback.
Arrays may be numpy (host) or torch CUDA tensors (device pointers are passed
through without copies).
"""
from __future__ import annotations

import ctypes as C
import os
import sys

# up to 17 concurrent streams per context (see pkrrgpu_create); must precede the
# process's CUDA context creation to take effect
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpkrr_gpu.so")

STRATEGIES = {"exact": 0, "dckrr": 1, "kkrr": 2, "kkrr2": 3, "kkrr3": 4, "bkrr": 5, "bkrr2": 6, "bkrr3": 7}
OK, INVALID, NPD, CUDA, LOGIC, IO = 0, 1, 2, 3, 4, 5

_d = C.POINTER(C.c_double)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)
_u8 = C.POINTER(C.c_uint8)


class NotPositiveDefinite(RuntimeError):
    """solver.hpp:17-21: a pivot was not strictly positive."""

    def __init__(self, pivot, msg=""):
        super().__init__(msg or f"matrix not positive definite: pivot {pivot}")
        self.pivot = int(pivot)


class CudaError(RuntimeError):
    pass


# pkrrgpu_allgather_fn: int (*)(void* user, void* dev_buf, int64_t bytes_per_rank)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64)
# pkrrgpu_bcast_fn: int (*)(void* user, void* dev_buf, int64_t bytes, int root)
BCAST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int)


class GridArgs(C.Structure):
    _fields_ = [("strategy", C.c_int), ("X_train", C.c_void_p), ("y_train", C.c_void_p), ("n", C.c_int64),
                ("d", C.c_int64), ("X_test", C.c_void_p), ("y_test", C.c_void_p), ("t", C.c_int64),
                ("X_eval", C.c_void_p), ("y_eval", C.c_void_p), ("t_eval", C.c_int64), ("p", C.c_int64),
                ("lambdas", C.c_void_p), ("n_lambdas", C.c_int64), ("sigmas", C.c_void_p),
                ("n_sigmas", C.c_int64), ("seed", C.c_uint64), ("km_threshold", C.c_double),
                ("km_max_iters", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("allgather", ALLGATHER_FN), ("allgather_user", C.c_void_p)]


class GridOut(C.Structure):
    _fields_ = [("cell_mse", C.c_void_p), ("cell_failed", C.c_void_p), ("cell_residual", C.c_void_p),
                ("cell_eval_mse", C.c_void_p), ("best_index", C.c_int64), ("part_sse", C.c_void_p),
                ("part_eval_sse", C.c_void_p), ("part_failed", C.c_void_p), ("part_residual", C.c_void_p),
                ("part_test_count", C.c_void_p), ("part_eval_count", C.c_void_p), ("part_of", C.c_void_p),
                ("centers", C.c_void_p), ("part_sizes", C.c_void_p), ("best_pred", C.c_void_p),
                ("best_eval_pred", C.c_void_p), ("p_effective", C.c_int64), ("flops_chol", C.c_double),
                ("flops_gram", C.c_double), ("flops_other", C.c_double), ("cell_pred", C.c_void_p),
                ("cell_eval_pred", C.c_void_p), ("pred_rows", C.c_int64)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libpkrr_gpu.so (built by build.py).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_1805_00569_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    sig = {
        "pkrrgpu_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
        "pkrrgpu_destroy": (None, [C.c_void_p]),
        "pkrrgpu_last_error": (C.c_char_p, []),
        "pkrrgpu_launch_count": (C.c_int64, [C.c_void_p]),
        "pkrrgpu_version": (C.c_char_p, []),
        "pkrrgpu_gram": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64,
                                   C.c_double, C.c_void_p]),
        "pkrrgpu_assemble": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_double, C.c_int64, C.c_void_p]),
        "pkrrgpu_cholesky": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, _i64]),
        "pkrrgpu_solve_spd": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
        "pkrrgpu_train_krr": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_double,
                                        C.c_double, C.c_void_p, _d, _i64]),
        "pkrrgpu_predict": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_double,
                                      C.c_void_p, C.c_int64, C.c_void_p]),
        "pkrrgpu_kmeans": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_uint64,
                                     C.c_double, C.c_int, C.c_void_p, C.c_void_p, _i64, C.POINTER(C.c_int)]),
        "pkrrgpu_kbalance": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_uint64,
                                       C.c_double, C.c_int, C.c_int, C.c_void_p, C.c_void_p, _i64]),
        "pkrrgpu_standardize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
        "pkrrgpu_auto_sigma_grid": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_uint64,
                                              C.c_void_p]),
        "pkrrgpu_load_libsvm": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
        "pkrrgpu_dataset_shape": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
        "pkrrgpu_dataset_csr": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
        "pkrrgpu_dataset_dense": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
        "pkrrgpu_dataset_free": (None, [C.c_void_p]),
        "pkrrgpu_nearest_center": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int64,
                                             C.c_void_p]),
        "pkrrgpu_make_partition": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                             C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, _i64]),
        "pkrrgpu_train_partitions": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                               C.c_int64, C.c_uint64, C.c_double, C.c_double,
                                               C.POINTER(C.c_void_p), _i64, _i64]),
        "pkrrgpu_models_count": (C.c_int64, [C.c_void_p]),
        "pkrrgpu_models_size": (C.c_int64, [C.c_void_p, C.c_int64]),
        "pkrrgpu_models_alpha": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
        "pkrrgpu_models_residual": (C.c_int, [C.c_void_p, C.c_int64, _d]),
        "pkrrgpu_models_free": (None, [C.c_void_p]),
        "pkrrgpu_predict_nearest": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
        "pkrrgpu_grid_search": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                          C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, _i64]),
        "pkrrgpu_grid_search_ex": (C.c_int, [C.c_void_p, C.POINTER(GridArgs), C.POINTER(GridOut)]),
        "pkrrgpu_last_timings": (C.c_int, [C.c_void_p, _d, C.c_int]),
        "pkrrgpu_stream": (C.c_void_p, [C.c_void_p]),
        "pkrrgpu_fp64_peak": (C.c_int, [C.c_void_p, _d]),
        "pkrrgpu_probe_potrf": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, _d]),
        "pkrrgpu_wait_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
        "pkrrgpu_train_parts": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                          C.c_void_p, C.c_int64, C.c_void_p, C.c_double, C.c_double,
                                          C.POINTER(C.c_void_p), _i64, _i64]),
        "pkrrgpu_device_count": (C.c_int, []),
        "pkrrgpu_models_import": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_double, C.POINTER(C.c_void_p)]),
        "pkrrgpu_models_predict": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                             C.c_void_p]),
        "pkrrgpu_models_centers": (C.c_int, [C.c_void_p, C.c_void_p]),
        "pkrrgpu_combine": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, _i64, C.c_void_p]),
        "pkrrgpu_multi_create": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
        "pkrrgpu_multi_destroy": (None, [C.c_void_p]),
        "pkrrgpu_multi_size": (C.c_int, [C.c_void_p]),
        "pkrrgpu_multi_context": (C.c_void_p, [C.c_void_p, C.c_int]),
        "pkrrgpu_multi_grid_search": (C.c_int, [C.c_void_p, C.POINTER(GridArgs), C.POINTER(GridOut)]),
        "pkrrgpu_multi_train_krr": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_double,
                                              C.c_double, C.c_void_p, _d, _i64]),
        "pkrrgpu_dist_train_krr": (C.c_int, [C.c_void_p, C.c_int, C.c_int, BCAST_FN, C.c_void_p, C.c_void_p,
                                             C.c_void_p, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_void_p,
                                             _d, _i64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    """Every entry point include/pkrr_gpu.h declares."""
    import re
    hdr = open(os.path.join(os.path.dirname(HERE), "include", "pkrr_gpu.h")).read()
    return sorted(set(re.findall(r"\b(pkrrgpu_[a-z_]+)\s*\(", hdr)))


def _check(rc, pivot=None):
    if rc == OK:
        return
    msg = _lib.pkrrgpu_last_error().decode()
    if rc == IO:
        raise RuntimeError(msg)
    if rc == NPD:
        raise NotPositiveDefinite(pivot if pivot is not None else -1, msg)
    if rc == INVALID:
        raise ValueError(msg)
    if rc == LOGIC:
        raise RuntimeError(msg)
    raise CudaError(msg)


def _ptr(a):
    """(pointer, keepalive) for numpy arrays or torch tensors (host or CUDA)."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            a = a.contiguous()
        return a.data_ptr(), a
    return a.ctypes.data, a


def _f64(a, device=None, dtype=np.float64):
    """An FP64 (or `dtype`) C-contiguous view the engine can read: numpy arrays are
    converted on the host; torch CUDA tensors are converted to `dtype` on the engine's
    device (a float32 tensor or a tensor on another GPU is never reinterpreted); torch
    CPU tensors become numpy arrays."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        import torch
        tdt = {np.float64: torch.float64, np.int32: torch.int32}[dtype]
        if a.is_cuda:
            dev = torch.device("cuda", a.device.index if device is None else device)
            return a.to(device=dev, dtype=tdt).contiguous()
        return np.ascontiguousarray(a.numpy(), dtype=dtype)
    return np.ascontiguousarray(a, dtype=dtype)


def _open_libsvm(path, threads=0):
    h = C.c_void_p()
    _check(load_library().pkrrgpu_load_libsvm(os.fsencode(path), int(threads), C.byref(h)))
    return h


def _shape(h):
    n, d, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    _check(_lib.pkrrgpu_dataset_shape(h, C.byref(n), C.byref(d), C.byref(nnz)))
    return n.value, d.value, nnz.value


def libsvm_csr(path, threads=0):
    """load_libsvm (dataset.cpp:83-125) on the host, no GPU needed: (row_ptr, col, val, y, d),
    the reference Dataset's CSR arrays."""
    h = _open_libsvm(path, threads)
    try:
        n, d, nnz = _shape(h)
        rp, col = np.empty(n + 1, np.int64), np.empty(nnz, np.int32)
        val, y = np.empty(nnz), np.empty(n)
        _check(_lib.pkrrgpu_dataset_csr(h, rp.ctypes.data, col.ctypes.data, val.ctypes.data, y.ctypes.data))
        return rp, col, val, y, d
    finally:
        _lib.pkrrgpu_dataset_free(h)


class Engine:
    """One engine per GPU (pkrrgpu_ctx).  One process per GPU for multi-GPU runs."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = C.c_void_p()
        _check(lib.pkrrgpu_create(device, C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_borrowed", False):  # a Group's context: the group destroys it
            self._h = None
        if getattr(self, "_h", None):
            _lib.pkrrgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _in(self, a, dtype=np.float64):
        """Caller array -> engine input.  A CUDA tensor may still be written by work
        queued on torch's current stream: the engine's launch stream is ordered after it
        (pkrrgpu_wait_stream) before any kernel reads the tensor."""
        a = _f64(a, self.device, dtype)
        if a is not None and hasattr(a, "data_ptr"):
            import torch
            _check(_lib.pkrrgpu_wait_stream(self._h, torch.cuda.current_stream(a.device).cuda_stream))
        return a

    @property
    def launches(self) -> int:
        return int(_lib.pkrrgpu_launch_count(self._h))

    @property
    def stream_handle(self) -> int:
        """cudaStream_t the engine launches on (wrap with torch.cuda.ExternalStream)."""
        return int(_lib.pkrrgpu_stream(self._h))

    def fp64_peak(self) -> float:
        v = C.c_double(0)
        _check(_lib.pkrrgpu_fp64_peak(self._h, C.byref(v)))
        return v.value

    def probe_potrf(self, m: int, alone: bool = False) -> dict:
        """Standalone factorization of an m x m system with events around every
        trailing-SYRK launch (the dominant kernel's live roofline); `alone` selects the
        panel schedule of a system factorised by itself (single-part grids)."""
        out = (C.c_double * 8)()
        _check(_lib.pkrrgpu_probe_potrf(self._h, int(m), 1 if alone else 0, out))
        return dict(total_ms=out[0], chol_flops=out[1], syrk_ms=out[2], syrk_flops=out[3],
                    syrk_launches=int(out[4]), npd=int(out[5]))

    def timings(self, parts: int = 0):
        n = 8 + 6 * parts
        ms = (C.c_double * n)()
        _lib.pkrrgpu_last_timings(self._h, ms, n)
        out = dict(partition=ms[0], train=ms[1], predict=ms[2], total=ms[3], cholesky=ms[4], gram=ms[5])
        if parts:
            out["part_chol_end_ms"] = [ms[8 + i] for i in range(parts)]
            # first cell, per part: gram start/end, Cholesky start/end, predict end (ms from the call start)
            out["part_timeline_ms"] = [[ms[8 + parts + 5 * i + j] for j in range(5)] for i in range(parts)]
        return out

    # ---- kernel.hpp ---------------------------------------------------------
    def gram(self, X, Y, sigma):
        X = self._in(X)
        same = Y is None or Y is X
        Y = X if same else self._in(Y)
        na, d = X.shape
        nb = Y.shape[0]
        K = np.empty((na, nb))
        px, kx = _ptr(X)
        py, ky = (px, kx) if same else _ptr(Y)
        _check(_lib.pkrrgpu_gram(self._h, px, na, py, nb, d, float(sigma), K.ctypes.data))
        return K

    def assemble_system(self, K, lam, m):
        K = self._in(K)
        A = np.empty_like(K)
        _check(_lib.pkrrgpu_assemble(self._h, K.ctypes.data, K.shape[0], float(lam), int(m), A.ctypes.data))
        return A

    # ---- solver.hpp ---------------------------------------------------------
    def cholesky(self, A):
        A = self._in(A)
        L = np.empty_like(A)
        piv = C.c_int64(-1)
        rc = _lib.pkrrgpu_cholesky(self._h, A.ctypes.data, A.shape[0], L.ctypes.data, C.byref(piv))
        _check(rc, piv.value)
        return L

    def solve_spd(self, L, b):
        L, b = self._in(L), self._in(b)
        x = np.empty(L.shape[0])
        _check(_lib.pkrrgpu_solve_spd(self._h, L.ctypes.data, L.shape[0], b.ctypes.data, x.ctypes.data))
        return x

    def train_krr(self, X, y, sigma, lam):
        X, y = self._in(X), self._in(y)
        m, d = X.shape
        alpha = np.empty(m)
        res = C.c_double(0)
        piv = C.c_int64(-1)
        px, kx = _ptr(X)
        py, ky = _ptr(y)
        rc = _lib.pkrrgpu_train_krr(self._h, px, py, m, d, float(sigma), float(lam), alpha.ctypes.data,
                                    C.byref(res), C.byref(piv))
        _check(rc, piv.value)
        return KrrModel(support=np.asarray(X) if not hasattr(X, "data_ptr") else X.cpu().numpy(),
                        alpha=alpha, sigma=float(sigma), lam=float(lam), residual_ratio=res.value, engine=self)

    def predict(self, S, alpha, sigma, Q):
        S, alpha, Q = self._in(S), self._in(alpha), self._in(Q)
        out = np.empty(Q.shape[0])
        _check(_lib.pkrrgpu_predict(self._h, S.ctypes.data, alpha.ctypes.data, S.shape[0], S.shape[1],
                                    float(sigma), Q.ctypes.data, Q.shape[0], out.ctypes.data))
        return out

    # ---- clustering.hpp -----------------------------------------------------
    def kmeans(self, X, k, seed, threshold=0.01, max_iters=100):
        X = self._in(X)
        n, d = X.shape
        mem = np.empty(n, np.int32)
        cen = np.empty((k, d))
        sz = np.empty(k, np.int64)
        it = C.c_int(0)
        px, kx = _ptr(X)
        _check(_lib.pkrrgpu_kmeans(self._h, px, n, d, k, seed, threshold, max_iters, mem.ctypes.data,
                                   cen.ctypes.data, sz.ctypes.data_as(_i64), C.byref(it)))
        return Clustering(k=k, centers=cen, membership=mem, sizes=sz, iterations=it.value)

    def kbalance(self, X, k, seed, threshold=0.01, max_iters=100, recompute_centers=True):
        X = self._in(X)
        n, d = X.shape
        mem = np.empty(n, np.int32)
        cen = np.empty((k, d))
        sz = np.empty(k, np.int64)
        px, kx = _ptr(X)
        _check(_lib.pkrrgpu_kbalance(self._h, px, n, d, k, seed, threshold, max_iters, int(recompute_centers),
                                     mem.ctypes.data, cen.ctypes.data, sz.ctypes.data_as(_i64)))
        return Clustering(k=k, centers=cen, membership=mem, sizes=sz)

    def nearest_center(self, centers, Q):
        centers, Q = self._in(centers), self._in(Q)
        single = Q.ndim == 1
        Q2 = Q.reshape(1, -1) if single else Q
        out = np.empty(Q2.shape[0], np.int32)
        _check(_lib.pkrrgpu_nearest_center(self._h, centers.ctypes.data, centers.shape[0], centers.shape[1],
                                           np.ascontiguousarray(Q2).ctypes.data, Q2.shape[0], out.ctypes.data))
        return int(out[0]) if single else out

    # ---- dataset.hpp: LIBSVM loader (dataset.cpp:83-125) ------------------------
    def load_libsvm(self, path, threads=0, device=False):
        """Dense (X, y) of a LIBSVM file: parsed by host threads into CSR, materialised
        in pinned staging, copied to numpy (or to CUDA tensors with device=True)."""
        h = _open_libsvm(path, threads)
        try:
            n, d, _ = _shape(h)
            if device:
                import torch
                X = torch.empty((n, d), dtype=torch.float64, device=f"cuda:{self.device}")
                y = torch.empty(n, dtype=torch.float64, device=f"cuda:{self.device}")
                _check(_lib.pkrrgpu_dataset_dense(self._h, h, X.data_ptr(), y.data_ptr()))
            else:
                X, y = np.empty((n, d)), np.empty(n)
                _check(_lib.pkrrgpu_dataset_dense(self._h, h, X.ctypes.data, y.ctypes.data))
            return X, y
        finally:
            _lib.pkrrgpu_dataset_free(h)

    # ---- dataset.hpp / strategies.hpp data preparation ------------------------
    def standardize(self, X_train, X_test=None):
        """dataset.cpp:199-232: (train_std, test_std, mean, stddev), bitwise the reference's."""
        X = self._in(X_train)
        n, d = X.shape
        T = np.zeros((0, d)) if X_test is None else self._in(X_test)
        tr, te = np.empty_like(X), np.empty_like(T)
        mean, sd = np.empty(d), np.empty(d)
        _check(_lib.pkrrgpu_standardize(self._h, X.ctypes.data, n, d, T.ctypes.data if T.size else None,
                                        T.shape[0], tr.ctypes.data, te.ctypes.data if T.size else None,
                                        mean.ctypes.data, sd.ctypes.data))
        return tr, te, mean, sd

    def auto_sigma_grid(self, X, seed):
        """strategies.cpp:204-234: the 9-point sigma grid around the median distance."""
        X = self._in(X)
        g = np.empty(9)
        _check(_lib.pkrrgpu_auto_sigma_grid(self._h, X.ctypes.data if X.size else None, X.shape[0],
                                            X.shape[1] if X.ndim == 2 else 0, int(seed), g.ctypes.data))
        return g

    # ---- strategies.hpp -----------------------------------------------------
    def make_partition(self, strategy, X, p, seed):
        X = self._in(X)
        n, d = X.shape
        part = np.empty(n, np.int32)
        order = np.empty(n, np.int64)
        cen = np.zeros((max(p, 1), d))
        pe = C.c_int64(0)
        px, kx = _ptr(X)
        _check(_lib.pkrrgpu_make_partition(self._h, STRATEGIES[strategy], px, n, d, p, seed, part.ctypes.data,
                                           order.ctypes.data, cen.ctypes.data, C.byref(pe)))
        pe = pe.value
        sizes = np.bincount(part, minlength=pe)
        parts, at = [], 0
        for t in range(pe):
            parts.append(order[at:at + sizes[t]].copy())
            at += sizes[t]
        has_c = STRATEGIES[strategy] not in (0, 1)
        return PartitionSet(p=pe, parts=parts, centers=cen[:pe] if has_c else None)

    def train_partitions(self, strategy, X, y, p, seed, sigma, lam):
        X, y = self._in(X), self._in(y)
        n, d = X.shape
        h = C.c_void_p()
        fp, piv = C.c_int64(-1), C.c_int64(-1)
        px, kx = _ptr(X)
        py, ky = _ptr(y)
        rc = _lib.pkrrgpu_train_partitions(self._h, STRATEGIES[strategy], px, py, n, d, p, seed, float(sigma),
                                           float(lam), C.byref(h), C.byref(fp), C.byref(piv))
        _check(rc, piv.value)
        return TrainedPartitions(self, h)

    def train_parts(self, X, y, parts, sigma, lam, centers=None):
        """train_partitions(ps, train, spec, lambda) with the caller's PartitionSet
        (strategies.cpp:104-133): `parts` = a list of row-index arrays (ps.parts, each in
        its own order) or a PartitionSet."""
        if isinstance(parts, PartitionSet):
            centers = parts.centers if centers is None else centers
            parts = parts.parts
        X, y = self._in(X), self._in(y)
        rows = np.ascontiguousarray(np.concatenate([np.asarray(q, np.int64) for q in parts]), np.int64)
        sizes = np.ascontiguousarray([len(q) for q in parts], np.int64)
        cen = self._in(centers) if centers is not None else None
        n, d = X.shape
        h = C.c_void_p()
        fp, piv = C.c_int64(-1), C.c_int64(-1)
        px, kx = _ptr(X)
        py, ky = _ptr(y)
        pc, kc = _ptr(cen)
        rc = _lib.pkrrgpu_train_parts(self._h, px, py, n, d, rows.ctypes.data, sizes.ctypes.data, len(parts), pc,
                                      float(sigma), float(lam), C.byref(h), C.byref(fp), C.byref(piv))
        _check(rc, piv.value)
        return TrainedPartitions(self, h)

    def dist_train_krr(self, X, y, sigma, lam, rank, world, bcast):
        """DKRR with one process per GPU (pkrrgpu_dist_train_krr): every rank calls it with
        the same inputs; bcast(dev_ptr, nbytes, root) broadcasts a device buffer (e.g.
        sharding.torch_broadcast).  Returns (alpha, residual) on every rank."""
        X = np.ascontiguousarray(X, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        alpha = np.empty(X.shape[0])
        res = C.c_double(0)
        piv = C.c_int64(-1)

        def _cb(user, buf, nbytes, root):
            try:
                bcast(int(buf), int(nbytes), int(root))
                return 0
            except Exception as exc:  # reported as a failed exchange by the engine
                print(f"pkrr broadcast failed: {exc!r}", file=sys.stderr)
                return 1
        cb = BCAST_FN(_cb)
        rc = _lib.pkrrgpu_dist_train_krr(self._h, int(rank), int(world), cb, None, X.ctypes.data, y.ctypes.data,
                                         X.shape[0], X.shape[1], float(sigma), float(lam), alpha.ctypes.data,
                                         C.byref(res), C.byref(piv))
        _check(rc, piv.value)
        return alpha, res.value

    def combine(self, strategy, p, pred, y, failed=None):
        """pkrrgpu_combine: cell combine + reference-order MSE + best cell over gathered
        per-cell predictions pred [ncell, P, t].  Returns (mse[ncell], best, best_pred)."""
        pred = np.ascontiguousarray(pred, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        nc, t = pred.shape[0], pred.shape[-1]
        fl = np.zeros(nc, np.uint8) if failed is None else np.ascontiguousarray(failed, np.uint8)
        mse_c = np.empty(nc)
        best = C.c_int64(-1)
        bp = np.zeros(t)
        _check(_lib.pkrrgpu_combine(self._h, STRATEGIES[strategy], int(p), t, nc, pred.ctypes.data, y.ctypes.data,
                                    fl.ctypes.data, mse_c.ctypes.data, C.byref(best), bp.ctypes.data))
        return mse_c, int(best.value), bp

    def grid_search(self, strategy, train_X, train_y, test_X, test_y, p, lambdas, sigmas, seed, *,
                    eval_X=None, eval_y=None, km_threshold=0.01, km_max_iters=0, rank=0, world=1,
                    want_partition=False, allgather=None, group=None):
        """strategies.cpp:343-507.  Returns GridResult (cells lambda-major).

        allgather (world > 1): fn(dev_ptr, bytes_per_rank) all-gathering a device buffer
        of `world` slices (sharding.torch_allgather / staged_allgather) -- shards the
        k-means partition over the ranks (bitwise the single-process partition)."""
        lam = np.ascontiguousarray(lambdas, np.float64)
        sig = np.ascontiguousarray(sigmas, np.float64)
        tX, ty, sX, sy = self._in(train_X), self._in(train_y), self._in(test_X), self._in(test_y)
        eX, ey = self._in(eval_X), self._in(eval_y)
        n, d = tX.shape
        t = sX.shape[0]
        te = 0 if eX is None else eX.shape[0]
        keep = []

        def P(a):
            p_, k_ = _ptr(a)
            keep.append(k_)
            return p_

        args = GridArgs(strategy=STRATEGIES[strategy], X_train=P(tX), y_train=P(ty), n=n, d=d, X_test=P(sX),
                        y_test=P(sy), t=t, X_eval=P(eX), y_eval=P(ey), t_eval=te, p=p,
                        lambdas=lam.ctypes.data, n_lambdas=lam.size, sigmas=sig.ctypes.data,
                        n_sigmas=sig.size, seed=seed, km_threshold=km_threshold, km_max_iters=km_max_iters,
                        rank=rank, world=world)
        if allgather is not None and world > 1:
            def _cb(user, buf, nbytes):
                try:
                    allgather(int(buf), int(nbytes))
                    return 0
                except Exception as exc:  # reported as a failed exchange by the engine
                    print(f"pkrr allgather failed: {exc!r}", file=sys.stderr)
                    return 1
            cb = ALLGATHER_FN(_cb)
            keep.append(cb)
            args.allgather = cb
        nc = lam.size * sig.size
        pmax = max(p, 1)
        res = dict(cell_mse=np.full(nc, np.nan), cell_failed=np.zeros(nc, np.uint8), cell_residual=np.zeros(nc),
                   cell_eval_mse=np.full(nc, np.nan), part_sse=np.zeros(nc * pmax),
                   part_eval_sse=np.zeros(nc * pmax), part_failed=np.zeros(nc * pmax, np.uint8),
                   part_residual=np.zeros(nc * pmax), part_test_count=np.zeros(pmax, np.int64),
                   part_eval_count=np.zeros(pmax, np.int64), part_sizes=np.zeros(pmax, np.int64),
                   best_pred=np.zeros(t), best_eval_pred=np.zeros(max(te, 1)),
                   cell_pred=np.zeros(nc * pmax * t), cell_eval_pred=np.zeros(nc * pmax * max(te, 1)))
        if want_partition:
            res["part_of"] = np.zeros(n, np.int32)
            res["centers"] = np.zeros((pmax, d))
        out = GridOut(**{k: v.ctypes.data for k, v in res.items()})
        if te == 0:
            out.cell_eval_pred = None
        if group is None:
            _check(_lib.pkrrgpu_grid_search_ex(self._h, C.byref(args), C.byref(out)))
        else:
            _check(_lib.pkrrgpu_multi_grid_search(group, C.byref(args), C.byref(out)))
        pe = out.p_effective
        P = out.pred_rows
        res["cell_pred"] = res["cell_pred"][: nc * P * t].reshape(nc, P, t)
        res["cell_eval_pred"] = res["cell_eval_pred"][: nc * P * te].reshape(nc, P, te) if te else None
        for k in ("part_sse", "part_eval_sse", "part_failed", "part_residual"):
            res[k] = res[k][: nc * pe].reshape(nc, pe)
        for k in ("part_test_count", "part_eval_count", "part_sizes"):
            res[k] = res[k][:pe]
        return GridResult(strategy=strategy, p=pe, lambdas=lam, sigmas=sig, best_index=int(out.best_index),
                          mse=res["cell_mse"], failed=res["cell_failed"].astype(bool),
                          residual=res["cell_residual"], eval_mse=res["cell_eval_mse"] if te else None,
                          best_pred=res["best_pred"], best_eval_pred=res["best_eval_pred"][:te] if te else None,
                          parts=res, flops=dict(chol=out.flops_chol, gram=out.flops_gram, other=out.flops_other))


class Group:
    """Several GPUs in ONE process (pkrrgpu_multi): one engine context and one host
    thread per device; grid_search shards the parts over the devices (LPT on m^3) and
    returns the one-context result bitwise.  A device may repeat (two contexts on one GPU)."""

    def __init__(self, devices):
        lib = load_library()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(lib.pkrrgpu_multi_create(devs, len(devices), C.byref(h)))
        self._h = h
        self.devices = list(devices)
        # engine facade on the first context (argument conversion, combine)
        self.first = Engine.__new__(Engine)
        self.first._borrowed = True
        self.first._h = C.c_void_p(lib.pkrrgpu_multi_context(h, 0))
        self.first.device = devices[0]

    def close(self):
        if getattr(self, "_h", None):
            self.first._h = None
            _lib.pkrrgpu_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return sum(int(_lib.pkrrgpu_launch_count(_lib.pkrrgpu_multi_context(self._h, i)))
                   for i in range(len(self.devices)))

    def train_krr(self, X, y, sigma, lam):
        """DKRR: train_krr (solver.cpp:89-125) of ONE system factorised across the group's
        GPUs (pkrrgpu_multi_train_krr).  Returns (alpha, residual)."""
        X = np.ascontiguousarray(X, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        alpha = np.empty(X.shape[0])
        res = C.c_double(0)
        piv = C.c_int64(-1)
        rc = _lib.pkrrgpu_multi_train_krr(self._h, X.ctypes.data, y.ctypes.data, X.shape[0], X.shape[1],
                                          float(sigma), float(lam), alpha.ctypes.data, C.byref(res), C.byref(piv))
        _check(rc, piv.value)
        return alpha, res.value

    def grid_search(self, strategy, train_X, train_y, test_X, test_y, p, lambdas, sigmas, seed, **kw):
        kw.pop("rank", None), kw.pop("world", None), kw.pop("allgather", None)
        return self.first.grid_search(strategy, train_X, train_y, test_X, test_y, p, lambdas, sigmas, seed,
                                      group=self._h, **kw)


@dataclass
class Clustering:
    k: int
    centers: np.ndarray
    membership: np.ndarray
    sizes: np.ndarray
    iterations: int = 0


@dataclass
class PartitionSet:
    p: int
    parts: list
    centers: object = None

    def has_centers(self):
        return self.centers is not None


@dataclass
class KrrModel:
    support: np.ndarray
    alpha: np.ndarray
    sigma: float
    lam: float
    residual_ratio: float
    engine: Engine = field(repr=False, default=None)

    def predict(self, Q):
        Q = np.asarray(Q, np.float64)
        single = Q.ndim == 1
        out = self.engine.predict(self.support, self.alpha, self.sigma, Q.reshape(1, -1) if single else Q)
        return float(out[0]) if single else out


class TrainedPartitions:
    """TrainedPartitions (strategies.hpp:44-47) resident on the GPU."""

    def __init__(self, engine: Engine, handle):
        self.engine = engine
        self._h = handle

    def __del__(self):
        try:
            if self._h:
                _lib.pkrrgpu_models_free(self._h)
                self._h = None
        except Exception:
            pass

    def __len__(self):
        return int(_lib.pkrrgpu_models_count(self._h))

    def alpha(self, t):
        a = np.empty(int(_lib.pkrrgpu_models_size(self._h, t)))
        _check(_lib.pkrrgpu_models_alpha(self._h, t, a.ctypes.data))
        return a

    def residual(self, t):
        r = C.c_double(0)
        _check(_lib.pkrrgpu_models_residual(self._h, t, C.byref(r)))
        return r.value

    def predict_nearest(self, Q):
        """strategies.cpp:142-149 batched: route by nearest_center, predict with that model."""
        Q = np.ascontiguousarray(Q, np.float64)
        out = np.empty(Q.shape[0])
        _check(_lib.pkrrgpu_predict_nearest(self.engine._h, self._h, Q.ctypes.data, Q.shape[0], out.ctypes.data))
        return out

    def predict(self, Q, part=-1):
        """KrrModel::predict (solver.cpp:74-87) of model `part`, or of every model
        ([p, q]) when part = -1."""
        Q = np.ascontiguousarray(Q, np.float64)
        rows = len(self) if part < 0 else 1
        out = np.empty((rows, Q.shape[0]))
        _check(_lib.pkrrgpu_models_predict(self.engine._h, self._h, int(part), Q.ctypes.data, Q.shape[0],
                                           out.ctypes.data))
        return out if part < 0 else out[0]

    def predict_average(self, Q):
        """strategies.cpp:135-140: sum of the models' predictions in model order / p."""
        pp = self.predict(Q)
        s = np.zeros(pp.shape[1])
        for row in pp:
            s = s + row
        return s / float(pp.shape[0])

    def predict_oracle(self, Q, y_true):
        """strategies.cpp:151-166: per row, the model prediction with the least squared
        error (first on ties).  Returns (predictions, chosen model)."""
        pp = self.predict(Q)
        err = (pp - np.asarray(y_true)[None, :]) ** 2
        best = np.zeros(pp.shape[1], np.int64)
        be = np.full(pp.shape[1], np.inf)
        for t in range(pp.shape[0]):
            better = err[t] < be
            be[better] = err[t][better]
            best[better] = t
        return pp[best, np.arange(pp.shape[1])], best

    def centers(self, d):
        c = np.empty((len(self), d))
        _check(_lib.pkrrgpu_models_centers(self._h, c.ctypes.data))
        return c


@dataclass
class GridResult:
    strategy: str
    p: int
    lambdas: np.ndarray
    sigmas: np.ndarray
    best_index: int
    mse: np.ndarray
    failed: np.ndarray
    residual: np.ndarray
    eval_mse: object = None
    best_pred: object = None
    best_eval_pred: object = None
    parts: dict = field(default_factory=dict, repr=False)
    flops: dict = field(default_factory=dict)

    def has_best(self):
        return self.best_index >= 0

    def max_residual(self):
        ok = ~self.failed
        return float(self.residual[ok].max()) if ok.any() else 0.0


def mse(pred, truth):
    """strategies.cpp:168-177 (host helper; the grid computes MSE on device)."""
    pred, truth = np.asarray(pred, np.float64), np.asarray(truth, np.float64)
    if pred.shape != truth.shape or pred.size == 0:
        raise ValueError("mse: length mismatch")
    s = 0.0
    for a, b in zip(pred, truth):
        s += (a - b) * (a - b)
    return s / pred.size
