"""CPU: the C-ABI library builds, loads and exports every symbol pkrr_gpu.h
declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import subprocess

import pytest

import paper_1805_00569_b200 as pk
from paper_1805_00569_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    path = build.build()
    lib = ctypes.CDLL(path)
    syms = pk.exported_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    lib = pk.load_library()
    assert lib.pkrrgpu_version().decode().startswith("pkrr-b200")


def test_no_oracle_in_product():
    # the product path must not import or link the test oracle
    # (the reference's "oracle" PREDICTOR, KKRR3 / predict_oracle, is product vocabulary;
    # the oracle PACKAGE / libraries are test infrastructure)
    import re
    pkg = os.path.join(ROOT, "paper_1805_00569_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), f
            assert "libpkrr_oracle" not in src and "libpkrr_ref" not in src and "oracle/" not in src, f
    out = subprocess.run(["ldd", pk.LIB_PATH], capture_output=True, text=True).stdout
    assert "pkrr_oracle" not in out and "pkrr_ref" not in out


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        pk.Engine(0)


def test_header_compiles_as_c():
    hdr = os.path.join(ROOT, "include", "pkrr_gpu.h")
    r = subprocess.run(["gcc", "-std=c99", "-fsyntax-only", "-x", "c", hdr], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
