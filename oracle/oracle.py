"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes loaders for the two CPU checkers:

* ``port()``      the plain-C restatement (oracle/levelset_oracle.c) -> oracle/_build/liblsoracle.so
* ``reference()`` the reference library compiled from its own sources
                  (oracle/Makefile) -> oracle/_ref/libref_levelset.so

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

from paper_2507_11542_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liblsoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_levelset.so")


def build(quiet=True):
    """Compile the restatement and (when /root/reference is present) the reference."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class OracleError(Exception):
    pass


def _raise(code, msg):
    if code == abi.EINVAL:
        raise ValueError(msg)
    if code == abi.ERANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


def _n(g):
    n = 1
    for d in range(g.dim):
        n *= g.counts[d]
    return n


class _Checker:
    """Same call surface over either library (prefix 'orc_' or 'ref_')."""

    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.path = path
        err = getattr(self.lib, prefix + "last_error")
        err.restype = C.c_char_p
        self._err = err

    def _call(self, name, *args):
        rc = getattr(self.lib, self.prefix + name)(*args)
        if rc != 0:
            _raise(rc, self._err().decode())

    # grid.cpp:50
    def axis(self, g, d):
        out = np.empty(g.counts[d], dtype=np.float64)
        if self.prefix == "orc_":
            self.lib.orc_axis(C.byref(g), C.c_int(d), abi.dptr(out))
        else:
            self._call("grid_axis", C.byref(g), C.c_int(d), abi.dptr(out))
        return out

    def pad_ghost(self, g, v, dim, width):
        v = np.ascontiguousarray(v, dtype=np.float64)
        n = g.counts[dim] if 0 <= dim < g.dim else 1
        out = np.empty(max(1, _n(g) // max(n, 1) * (n + 2 * max(width, 0))), dtype=np.float64)
        self._call("pad_ghost", C.byref(g), abi.dptr(v), C.c_int(dim), C.c_int(width), abi.dptr(out))
        return out

    def shift_along_dim(self, g, padded, dim, width, offset):
        padded = np.ascontiguousarray(padded, dtype=np.float64)
        out = np.empty(_n(g), dtype=np.float64)
        self._call("shift_along_dim", C.byref(g), abi.dptr(padded), C.c_int(dim), C.c_int(width),
                   C.c_int(offset), abi.dptr(out))
        return out

    def upwind(self, g, v, dim, scheme):
        v = np.ascontiguousarray(v, dtype=np.float64)
        L = np.empty(_n(g), dtype=np.float64)
        R = np.empty(_n(g), dtype=np.float64)
        self._call("upwind", C.byref(g), abi.dptr(v), C.c_int(dim), C.c_int(scheme), abi.dptr(L), abi.dptr(R))
        return L, R

    def term_lf(self, g, p, t, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty(_n(g), dtype=np.float64)
        b = C.c_double()
        self._call("term_lf", C.byref(g), C.byref(p), C.c_double(t), abi.dptr(v), abi.dptr(out), C.byref(b))
        return out, b.value

    def restrict_update(self, dvdt, direction):
        dvdt = np.ascontiguousarray(dvdt, dtype=np.float64)
        out = np.empty_like(dvdt)
        self._call("restrict_update", C.c_size_t(dvdt.size), abi.dptr(dvdt), C.c_int(direction), abi.dptr(out))
        return out

    def integrate(self, g, p, method, t0, tf, v0, opts=None, log_cap=1 << 16):
        v = np.array(v0, dtype=np.float64, copy=True)
        log = (abi.LsgStepLog * log_cap)()
        n = C.c_size_t()
        tfin = C.c_double()
        self._call("integrate", C.byref(g), C.byref(p), C.c_int(method), C.c_double(t0), C.c_double(tf),
                   abi.dptr(v), C.byref(opts) if opts is not None else None, log, C.c_size_t(log_cap),
                   C.byref(n), C.byref(tfin))
        steps = np.array([[e.t, e.dt, e.step_bound, e.v_min, e.v_max] for e in log[: min(n.value, log_cap)]],
                         dtype=np.float64).reshape(-1, 5)
        return v, steps, tfin.value

    def solve_brt(self, g, p, v0, tspan, n_checkpoints, method=abi.CFL3, opts=None, log_cap=1 << 16):
        v0 = np.ascontiguousarray(v0, dtype=np.float64)
        N = _n(g)
        ck = np.empty(max(1, n_checkpoints) * N, dtype=np.float64)
        times = np.empty(max(1, n_checkpoints), dtype=np.float64)
        n_out = C.c_int()
        log = (abi.LsgStepLog * log_cap)()
        n = C.c_size_t()
        args = [C.byref(g), C.byref(p), abi.dptr(v0), C.c_double(tspan[0]), C.c_double(tspan[1]),
                C.c_int(n_checkpoints), C.c_int(method), C.byref(opts) if opts is not None else None,
                abi.dptr(ck), abi.dptr(times), C.byref(n_out), log, C.c_size_t(log_cap), C.byref(n)]
        if self.prefix == "ref_":
            args.append(None)
        self._call("solve_brt", *args)
        k = n_out.value
        steps = np.array([[e.t, e.dt, e.step_bound, e.v_min, e.v_max] for e in log[: min(n.value, log_cap)]],
                         dtype=np.float64).reshape(-1, 5)
        return ck[: k * N].reshape(k, N), times[:k].copy(), steps

    def sphere(self, g, center, radius):
        out = np.empty(_n(g), dtype=np.float64)
        c = np.ascontiguousarray(center, dtype=np.float64)
        self._call("sphere", C.byref(g), abi.dptr(c), C.c_double(radius), abi.dptr(out))
        return out

    def cylinder(self, g, ignored_dims, center, radius):
        out = np.empty(_n(g), dtype=np.float64)
        c = np.ascontiguousarray(center, dtype=np.float64)
        mask = 0
        for d in ignored_dims:
            mask |= 1 << d
        self._call("cylinder", C.byref(g), C.c_uint(mask), abi.dptr(c), C.c_double(radius), abi.dptr(out))
        return out


    def rectangle(self, g, lower, upper):
        out = np.empty(_n(g), dtype=np.float64)
        lo = np.ascontiguousarray(lower, dtype=np.float64)
        up = np.ascontiguousarray(upper, dtype=np.float64)
        self._call("rectangle", C.byref(g), abi.dptr(lo), abi.dptr(up), abi.dptr(out))
        return out

    def ellipsoid(self, g, radius):
        out = np.empty(_n(g), dtype=np.float64)
        self._call("ellipsoid", C.byref(g), C.c_double(radius), abi.dptr(out))
        return out

    def set_op(self, g, op, a, b=None):
        out = np.empty(_n(g), dtype=np.float64)
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = a if b is None else np.ascontiguousarray(b, dtype=np.float64)
        self._call("set_op", C.byref(g), C.c_int(op), abi.dptr(a), abi.dptr(b), abi.dptr(out))
        return out


class _Reference(_Checker):
    def solve_rockets(self, n, tspan, n_checkpoints, theta_periodic=False, log_cap=1 << 16):
        N = n ** 3
        v = np.empty(N, dtype=np.float64)
        log = (abi.LsgStepLog * log_cap)()
        cnt = C.c_size_t()
        self._call("solve_rockets", C.c_int(n), C.c_int(1 if theta_periodic else 0), C.c_double(tspan[0]),
                   C.c_double(tspan[1]), C.c_int(n_checkpoints), abi.dptr(v), log, C.c_size_t(log_cap),
                   C.byref(cnt))
        steps = np.array([[e.t, e.dt, e.step_bound, e.v_min, e.v_max] for e in log[: min(cnt.value, log_cap)]],
                         dtype=np.float64).reshape(-1, 5)
        return v, steps

    def rocket_plugins(self, g, params5, costate):
        """reachability.cpp rocket_hamiltonian / rocket_dissipation on given fields."""
        n = _n(g)
        h, b0, b1, b2 = (np.empty(n) for _ in range(4))
        prm = np.ascontiguousarray(params5, dtype=np.float64)
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in costate]
        self._call("rocket_plugins", C.byref(g), abi.dptr(prm), abi.dptr(cs[0]), abi.dptr(cs[1]), abi.dptr(cs[2]),
                   abi.dptr(h), abi.dptr(b0), abi.dptr(b1), abi.dptr(b2))
        return h, [b0, b1, b2]

    def rocket_initial(self, n, theta_periodic=False):
        v = np.empty(n ** 3, dtype=np.float64)
        self._call("rocket_initial", C.c_int(n), C.c_int(1 if theta_periodic else 0), abi.dptr(v))
        return v

    def bench(self, g, p, method, v0, tf, opts=None, nthreads=1):
        """Wall seconds for `nthreads` concurrent replicas of integrate(...), steps per replica."""
        v0 = np.ascontiguousarray(v0, dtype=np.float64)
        secs = C.c_double()
        steps = C.c_size_t()
        self._call("bench", C.byref(g), C.byref(p), C.c_int(method), abi.dptr(v0), C.c_double(tf),
                   C.byref(opts) if opts is not None else None, C.c_int(nthreads), C.byref(secs), C.byref(steps))
        return secs.value, steps.value


_cache = {}


def port():
    if "port" not in _cache:
        _cache["port"] = _Checker(PORT_SO, "orc_")
    return _cache["port"]


def reference():
    if "ref" not in _cache:
        _cache["ref"] = _Reference(REF_SO, "ref_")
    return _cache["ref"]


def have_reference():
    return os.path.exists(REF_SO)


INF = math.inf
