"""ctypes mirror of include/lsg.h (descriptors, enums and status codes).

Shared by the product binding (``_lib.py``) and the test-side oracle loader;
it holds no behaviour of its own.
"""
from __future__ import annotations

import ctypes as C
import math

MAX_DIM = 6
MAX_PARAMS = 16

OK, EINVAL, ERANGE, ENUMERIC, ECUDA, ENCCL, ENOMEM = range(7)

BC_PERIODIC, BC_EXTRAPOLATE = 0, 1
SCHEME_FIRST, SCHEME_ENO2, SCHEME_ENO3, SCHEME_WENO5 = 0, 1, 2, 3
GROW, SHRINK = 0, 1
CFL1, CFL2, CFL3 = 0, 1, 2

HAM_LINEAR, HAM_ROTATION, HAM_ROCKETS, HAM_AIR3D, HAM_DBLINT4, HAM_DUBINS6, HAM_NORMAL = range(1, 8)
HAM_NAMES = {
    HAM_LINEAR: "linear",
    HAM_ROTATION: "rotation",
    HAM_ROCKETS: "rockets",
    HAM_AIR3D: "air3d",
    HAM_DBLINT4: "dblint4",
    HAM_DUBINS6: "dubins6",
    HAM_NORMAL: "normal",
}


class LsgGrid(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("counts", C.c_int * MAX_DIM),
        ("mins", C.c_double * MAX_DIM),
        ("maxs", C.c_double * MAX_DIM),
        ("periodic_mask", C.c_uint),
    ]


class LsgProblem(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("scheme", C.c_int),
        ("direction", C.c_int),
        ("restrict_update", C.c_int),
        ("options", C.c_int),
        ("params", C.c_double * MAX_PARAMS),
    ]


class LsgOpts(C.Structure):
    _fields_ = [
        ("cfl_factor", C.c_double),
        ("max_step", C.c_double),
        ("termination_epsilon", C.c_double),
        ("checkpoint_times", C.POINTER(C.c_double)),
        ("n_checkpoint_times", C.c_size_t),
    ]


class LsgStepLog(C.Structure):
    _fields_ = [
        ("t", C.c_double),
        ("dt", C.c_double),
        ("step_bound", C.c_double),
        ("v_min", C.c_double),
        ("v_max", C.c_double),
    ]


def make_grid(mins, maxs, counts, periodic_dims=()) -> LsgGrid:
    g = LsgGrid()
    g.dim = len(counts)
    if not (len(mins) == len(maxs) == len(counts)):
        # the library reports the reference's message; keep the struct consistent
        g.dim = -1
        return g
    for d in range(min(len(counts), MAX_DIM)):
        g.counts[d] = int(counts[d])
        g.mins[d] = float(mins[d])
        g.maxs[d] = float(maxs[d])
    mask = 0
    for d in periodic_dims:
        mask |= 1 << int(d) if 0 <= int(d) < 32 else 1 << 31
    g.periodic_mask = mask
    return g


OPT_WENO5_FAST = 1


def make_problem(kind, scheme, params=(), direction=GROW, restrict_update=False, options=0) -> LsgProblem:
    p = LsgProblem()
    p.options = int(options)
    p.kind = int(kind)
    p.scheme = int(scheme)
    p.direction = int(direction)
    p.restrict_update = 1 if restrict_update else 0
    for k, val in enumerate(params):
        p.params[k] = float(val)
    return p


def linear_params(c, bounds=None, offset=0.0):
    """params for HAM_LINEAR: c_d at [0..5], bound_d at [6..11], offset at [12]."""
    prm = [0.0] * MAX_PARAMS
    for d, cd in enumerate(c):
        prm[d] = float(cd)
        prm[6 + d] = abs(float(cd)) if bounds is None else float(bounds[d])
    prm[12] = float(offset)
    return prm


def make_opts(cfl_factor=0.32, max_step=math.inf, termination_epsilon=1e-6, checkpoint_times=()):
    o = LsgOpts()
    o.cfl_factor = cfl_factor
    o.max_step = max_step
    o.termination_epsilon = termination_epsilon
    ck = list(checkpoint_times)
    if ck:
        arr = (C.c_double * len(ck))(*ck)
        o.checkpoint_times = arr
        o.n_checkpoint_times = len(ck)
        o._keep = arr  # keep the buffer alive with the struct
    else:
        o.checkpoint_times = None
        o.n_checkpoint_times = 0
    return o


def dptr(a):
    """numpy float64 array -> c_double pointer (array must be C-contiguous)."""
    return a.ctypes.data_as(C.POINTER(C.c_double))
