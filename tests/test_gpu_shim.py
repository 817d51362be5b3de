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


def test_cpp_dropin_reference_benchmark_outputs():
    """The reference's own microbenchmark suite (benchmarks/bench_kernels.cpp,
    from proj/benchmarks/bench_kernels.cpp) built against the drop-in: every
    case's output checksum equals the reference build's bit for bit
    (tests/golden/bench_kernels_checksums.json)."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    binary = os.path.join(root, "benchmarks", "bench_kernels_b200")
    assert os.path.exists(binary), "benchmarks/bench_kernels_b200 not built: run __graft_entry__.build()"
    out = subprocess.run([binary, "--large", "--min-time", "0"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    got = {r["name"]: r["checksum"] for r in map(json.loads, filter(None, out.stdout.splitlines()))}
    want = json.load(open(os.path.join(root, "tests", "golden", "bench_kernels_checksums.json")))["checksums"]
    assert set(got) == set(want)
    bad = {k: (got[k], want[k]) for k in want if got[k] != want[k]}
    assert not bad, bad


def test_divmod_index_exact():
    """The generic kernel's index decomposition (divmod_index, lsg_device.cuh)
    equals exact 64-bit integer division on ~1e8 inputs up to 2^40, dense
    around multiples of every divisor 1..65536 (tests/cpp/divmod_check.cu)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    binary = os.path.join(root, "tests", "cpp", "divmod_check")
    assert os.path.exists(binary), "tests/cpp/divmod_check not built: run __graft_entry__.build()"
    out = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "divmod ok" in out.stdout


@pytest.mark.gpu
def test_weno5_exact_blocks_bitwise():
    """The exact WENO5's select-free constant divisions and the shared-quotient
    two-node form (line_lr2<WENO5>) equal the reference's IEEE arithmetic bit
    for bit on ~1e9 random operands and ~2e8 random windows, including zeros,
    flat runs, subnormal-adjacent and overflowing differences
    (tests/cpp/weno5_check.cu; spatial_derivatives.cpp:78-97)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    binary = os.path.join(root, "tests", "cpp", "weno5_check")
    assert os.path.exists(binary), "tests/cpp/weno5_check not built: run __graft_entry__.build()"
    out = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "weno5 ok" in out.stdout
