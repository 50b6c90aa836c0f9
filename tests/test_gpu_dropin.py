"""The C++ drop-in (include/fpr/pagerank_b200.hpp) at a reference-shaped call
site: the reference's generate_rmat/build_csr/build_layout + engines next to
fpr::pagerank_{ec,fused}_b200 (binary built by tests/cpp/Makefile)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "build", "test_dropin")


def test_cpp_dropin():
    if not os.path.exists(BIN):
        pytest.skip("drop-in binary not built (needs the reference headers at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("OK")
