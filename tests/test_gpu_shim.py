"""The reference's doctest cases re-expressed against the C++ drop-in layer
(include/levelset_b200/levelset.hpp -> liblevelset_b200.so -> liblsg_b200.so),
compiled by build() into tests/cpp/shim_tests and run on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "shim_tests")


def test_cpp_dropin_reference_cases():
    assert os.path.exists(BIN), "tests/cpp/shim_tests not built: run __graft_entry__.build()"
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout
