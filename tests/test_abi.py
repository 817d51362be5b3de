"""CPU tests of the C-ABI boundary: the library loads, exports every symbol
include/lsg.h declares, and its host-only entry points (grid validation and
geometry, Grid::create semantics grid.cpp:9-66) behave like the reference.
No compute call is made here (there is no GPU in the build container)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from paper_2507_11542_b200 import _lib, abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "lsg.h")).read()
    return sorted(set(re.findall(r"\b(lsg_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.lsg_abi_version() == 1


def test_shim_library_exports():
    path = os.path.join(ROOT, "paper_2507_11542_b200", "liblevelset_b200.so")
    if not os.path.exists(path):
        pytest.skip("C++ drop-in layer not built")
    C.CDLL(_lib.LIB_PATH, mode=C.RTLD_GLOBAL)
    C.CDLL(path)


def test_grid_check_mirrors_grid_create():
    lib = _lib.load()
    ok = abi.make_grid([0.0, -1.0], [1.0, 1.0], [5, 7], [1])
    assert lib.lsg_grid_check(C.byref(ok)) == abi.OK
    bad = [
        abi.make_grid([0.0], [1.0], [2]),            # counts >= 3 (grid.cpp:19)
        abi.make_grid([1.0], [1.0], [5]),            # max > min (grid.cpp:21)
        abi.make_grid([0.0], [1.0], [5], [1]),       # periodic dim in range (grid.cpp:24)
        abi.make_grid([], [], []),                   # dim >= 1 (grid.cpp:14)
    ]
    for g in bad:
        with pytest.raises(ValueError):
            _lib.call("lsg_grid_check", C.byref(g))


def test_grid_geometry():
    g = abi.make_grid([-64.0, -1.0], [64.0, 2.0], [50, 7])
    dx = C.c_double()
    _lib.call("lsg_grid_spacing", C.byref(g), 0, C.byref(dx))
    assert dx.value == (64.0 - -64.0) / 49.0
    n = C.c_size_t()
    _lib.call("lsg_grid_node_count", C.byref(g), C.byref(n))
    assert n.value == 350
    ax = np.empty(50)
    _lib.call("lsg_grid_axis", C.byref(g), 0, abi.dptr(ax))
    assert np.array_equal(ax, -64.0 + np.arange(50) * ((64.0 + 64.0) / 49.0))


def test_opts_default_mirrors_integrator_options():
    o = abi.LsgOpts()
    _lib.load().lsg_opts_default(C.byref(o))
    assert o.cfl_factor == 0.32 and o.max_step == math.inf and o.termination_epsilon == 1e-6


def test_no_cpu_fallback_without_device():
    """Without a GPU every compute path fails loudly (LSG_ECUDA)."""
    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        _lib.Context(0)


def test_null_solver_handles_are_rejected():
    """Every solver entry point returns LSG_EINVAL for a null handle (no crash,
    no device needed)."""
    lib = _lib.load()
    d, p, n, sz = C.c_double(), C.c_void_p(), C.c_int(), C.c_size_t()
    buf = (C.c_double * 4)()
    calls = [
        ("lsg_solver_set_field", (None, buf)),
        ("lsg_solver_get_field", (None, buf)),
        ("lsg_solver_set_field_device", (None, buf)),
        ("lsg_solver_field_device", (None, C.byref(p))),
        ("lsg_solver_init_shape", (None, 0, 0, None, C.c_double(1.0))),
        ("lsg_solver_step_bound", (None, C.c_double(0.0), C.byref(d))),
        ("lsg_solver_step", (None, C.c_double(0.0), C.c_double(0.01))),
        ("lsg_solver_step_host", (None, C.c_double(0.0), C.c_double(0.01), buf, buf)),
        ("lsg_solver_step_timed", (None, C.c_double(0.0), C.c_double(0.01), buf, buf)),
        ("lsg_solver_integrate", (None, C.c_double(0.0), C.c_double(1.0), None, None, C.c_size_t(0), C.byref(sz),
                                  C.byref(d))),
        ("lsg_solver_write_snapshot", (None, C.c_double(0.0), b"/tmp/x")),
        ("lsg_solver_stream", (None, C.byref(p))),
        ("lsg_solver_launches_per_step", (None, C.byref(n))),
        ("lsg_solver_slab", (None, C.byref(n), C.byref(n), C.byref(sz))),
    ]
    for name, args in calls:
        assert getattr(lib, name)(*args) == abi.EINVAL, name
    assert lib.lsg_solver_destroy(None) == abi.OK
