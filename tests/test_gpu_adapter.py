"""GPU: the C++ drop-in adapter (include/pkrr_gpu.hpp) against the reference
library itself, through tests/_bin/test_adapter (built by tests/cpp/Makefile in
the build container, where /root/reference headers exist)."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(__file__), "_bin", "test_adapter")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="tests/_bin/test_adapter not built")
def test_cpp_adapter_against_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
