"""LIBSVM loader: host-side, multi-threaded parse into the
reference Dataset's CSR arrays -- checked bitwise against the reference's own
load_libsvm (dataset.cpp:83-125, through oracle/_ref), including its error messages.
CPU tests; the dense pinned-staging path is checked on the GPU."""
import os

import numpy as np
import pytest

import paper_1805_00569_b200 as pk
from oracle import Reference


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


def _random_file(rng, n, d, density, crlf=False, trailing_newline=True):
    lines = []
    for i in range(n):
        if i % 97 == 13:
            lines.append("   ")  # blank line: skipped
        nnz = rng.binomial(d, density)
        idx = np.sort(rng.choice(d, size=nnz, replace=False)) + 1
        vals = rng.standard_normal(nnz) * 10.0 ** rng.integers(-3, 4, nnz)
        lab = rng.standard_normal()
        sep = "\t" if i % 5 == 0 else " "
        feats = sep.join(f"{j}:{float(v)!r}" if i % 3 else f"{j}:{float(v):.6e}" for j, v in zip(idx, vals))
        lines.append(f"{float(lab)!r}{sep}{feats}" if nnz else f"{float(lab):.17g}")
    eol = "\r\n" if crlf else "\n"
    return eol.join(lines) + (eol if trailing_newline else "")


needs_ref = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("n,d,density,crlf,trail,threads", [
    (1, 3, 1.0, False, False, 0), (50, 8, 0.5, False, True, 1), (300, 20, 0.3, True, True, 0),
    (20000, 90, 0.8, False, False, 0), (20000, 90, 0.8, False, True, 7)])
def test_csr_bitwise_equals_reference(tmp_path, n, d, density, crlf, trail, threads):
    rng = np.random.default_rng(n + d)
    path = _write(tmp_path, "a.svm", _random_file(rng, n, d, density, crlf, trail))
    got = pk.libsvm_csr(path, threads)
    ref = Reference().load_libsvm(path)
    for a, b in zip(got[:4], ref[:4]):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    assert got[4] == ref[4]


@needs_ref
@pytest.mark.parametrize("text", [
    "1 2:3\nabc 1:2\n", "1 0:1\n", "1 3:1 2:1\n", "1 1:x\n", "1 1 2\n", "\n\n  \n",
    "1 1:1\n2 1:1 1:2\n3 5:1\n" * 3000])
def test_errors_match_reference(tmp_path, text):
    path = _write(tmp_path, "bad.svm", text)
    with pytest.raises(RuntimeError) as ours:
        pk.libsvm_csr(path)
    with pytest.raises(RuntimeError) as ref:
        Reference().load_libsvm(path)
    assert str(ours.value) == str(ref.value)


def test_missing_file_raises():
    with pytest.raises(RuntimeError, match="cannot open"):
        pk.libsvm_csr("/nonexistent/file.svm")


@pytest.mark.gpu
def test_dense_staging(tmp_path, engine):
    rng = np.random.default_rng(3)
    path = _write(tmp_path, "c.svm", _random_file(rng, 5000, 40, 0.4))
    rp, col, val, y, d = pk.libsvm_csr(path)
    dense = np.zeros((len(y), d))
    for i in range(len(y)):
        dense[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    X, yy = engine.load_libsvm(path)
    assert np.array_equal(X, dense) and np.array_equal(yy, y)
    Xd, yd = engine.load_libsvm(path, device=True)
    assert np.array_equal(Xd.cpu().numpy(), dense) and np.array_equal(yd.cpu().numpy(), y)
