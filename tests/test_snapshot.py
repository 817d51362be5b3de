"""Checkpoint files in the reference's snapshot format (snapshot.cpp:69-129),
written by the product's C ABI (host-only code) and by the reference itself
(oracle/_ref): byte-identical files, cross-readable."""
import os

import numpy as np
import pytest

from conftest import assert_bitwise
from paper_2507_11542_b200 import _lib, abi
import helpers as H


@pytest.mark.parametrize("grid", [
    abi.make_grid([-64.0, -64.0, -1.5707963267948966], [64.0, 64.0, 1.4], [9, 7, 5], (2,)),
    abi.make_grid([0.1], [1.0 / 3.0], [11]),
    abi.make_grid([-1.0] * 4, [1.0] * 4, [3, 4, 5, 3]),
])
def test_snapshot_matches_reference_bytes(ref, tmp_path, grid):
    v = H.random_field(grid, 3, -1e3, 1e3)
    ours, theirs = tmp_path / "ours.bin", tmp_path / "ref.bin"
    _lib.write_snapshot(grid, v, 0.1 + 0.2, ours)
    ref_t = __import__("ctypes")
    import ctypes as C
    rc = ref.lib.ref_write_snapshot(C.byref(grid), abi.dptr(np.ascontiguousarray(v)), C.c_double(0.1 + 0.2),
                                    str(theirs).encode())
    assert rc == 0
    assert ours.read_bytes() == theirs.read_bytes()
    g2, v2, t2 = _lib.read_snapshot(theirs)
    assert t2 == 0.1 + 0.2 and g2.dim == grid.dim
    for d in range(grid.dim):
        assert g2.counts[d] == grid.counts[d] and g2.mins[d] == grid.mins[d] and g2.maxs[d] == grid.maxs[d]
    assert_bitwise(v2, v, "payload")


def test_snapshot_errors(tmp_path):
    g = abi.make_grid([0.0], [1.0], [5])
    p = tmp_path / "s.bin"
    _lib.write_snapshot(g, np.arange(5.0), 1.0, p)
    data = p.read_bytes()
    (tmp_path / "short.bin").write_bytes(data[:-8])
    with pytest.raises(RuntimeError, match="truncated"):
        _lib.read_snapshot(tmp_path / "short.bin")
    (tmp_path / "bad.bin").write_bytes(b"dimz 1\n" + data[7:])
    with pytest.raises(RuntimeError, match="expected header line"):
        _lib.read_snapshot(tmp_path / "bad.bin")
    nan = np.arange(5.0)
    nan[2] = np.nan
    _lib.write_snapshot(g, nan, 1.0, tmp_path / "nan.bin")
    with pytest.raises(RuntimeError, match="non-finite"):
        _lib.read_snapshot(tmp_path / "nan.bin")
