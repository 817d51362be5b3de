"""ctypes binding of the C ABI in include/lsg.h (liblsg_b200.so).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2507_11542_b200/csrc``).  There is no CPU fallback: if the
library is missing this module raises on load, and every compute call raises
``RuntimeError`` when no CUDA device is usable.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import weakref

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
# LSG_LIB=checked selects the bounds-checked build (make -C csrc checked; tools/checked_run.sh),
# LSG_LIB=<name> the in-tree liblsg_b200_<name>.so (A/B of two builds on one box)
LIB_PATH = os.path.join(HERE, "liblsg_b200_%s.so" % os.environ["LSG_LIB"] if os.environ.get("LSG_LIB") else "liblsg_b200.so")

# every symbol include/lsg.h declares
EXPORTS = (
    "lsg_abi_version", "lsg_last_error", "lsg_opts_default", "lsg_device_count",
    "lsg_ctx_create", "lsg_nccl_unique_id", "lsg_ctx_create_dist", "lsg_ctx_destroy",
    "lsg_ctx_synchronize", "lsg_ctx_launch_count", "lsg_host_alloc", "lsg_host_free",
    "lsg_grid_check", "lsg_grid_spacing", "lsg_grid_node_count", "lsg_grid_axis", "lsg_slab_partition",
    "lsg_pad_ghost", "lsg_shift_along_dim", "lsg_upwind", "lsg_term_lf", "lsg_restrict_update", "lsg_set_op",
    "lsg_eval_hamiltonian", "lsg_eval_dissipation",
    "lsg_integrate", "lsg_solve_brt", "lsg_write_snapshot", "lsg_read_snapshot",
    "lsg_extract_zero_set_2d", "lsg_slice_2d",
    "lsg_solver_create", "lsg_solver_create_slabs", "lsg_solver_destroy", "lsg_solver_slab",
    "lsg_solver_set_field", "lsg_solver_get_field", "lsg_solver_set_field_device",
    "lsg_solver_field_device", "lsg_solver_init_shape", "lsg_solver_apply_shape", "lsg_solver_complement",
    "lsg_solver_step_bound", "lsg_solver_step",
    "lsg_solver_step_host",
    "lsg_solver_step_timed",
    "lsg_solver_integrate", "lsg_solver_write_snapshot", "lsg_solver_stream", "lsg_solver_launches_per_step",
    "lsg_probe_fp64_rate", "lsg_ctx_comm_info", "lsg_gather_field", "lsg_halo_plan",
    "lsg_solve_brt_resume",
)

_lib = None


def load():
    """Load liblsg_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        lib.lsg_last_error.restype = C.c_char_p
        lib.lsg_abi_version.restype = C.c_int
        _lib = lib
    return _lib


def raise_for(rc):
    if rc == abi.OK:
        return
    msg = load().lsg_last_error().decode()
    if rc == abi.EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == abi.ERANGE:
        raise IndexError(msg)  # std::out_of_range
    raise RuntimeError(msg)  # std::runtime_error / device faults


def call(name, *args):
    raise_for(getattr(load(), name)(*args))


def node_count(g):
    n = 1
    for d in range(g.dim):
        n *= g.counts[d]
    return n


def _steps(log, n, cap):
    return np.array([[e.t, e.dt, e.step_bound, e.v_min, e.v_max] for e in log[: min(n, cap)]],
                    dtype=np.float64).reshape(-1, 5)


_live_contexts = weakref.WeakSet()


@atexit.register
def _close_all():
    """Destroy solvers before their contexts while the runtime is intact (the
    interpreter's teardown order would otherwise be arbitrary)."""
    for ctx in list(_live_contexts):
        try:
            ctx.close()
        except Exception:
            pass


class Context:
    """One CUDA device + stream (lsg_ctx).  Closing it closes its solvers first."""

    def __init__(self, device=0, rank=0, nranks=1, nccl_id=None):
        self.h = None
        self._solvers = weakref.WeakSet()
        h = C.c_void_p()
        if nranks > 1 or nccl_id is not None:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("distributed context needs the 128-byte NCCL unique id")
            buf = (C.c_ubyte * 128).from_buffer_copy(bytes(nccl_id))
            call("lsg_ctx_create_dist", C.c_int(device), C.c_int(rank), C.c_int(nranks), buf, C.byref(h))
        else:
            call("lsg_ctx_create", C.c_int(device), C.byref(h))
        self.h = h
        self.device, self.rank, self.nranks = device, rank, nranks
        _live_contexts.add(self)

    def close(self):
        if self.h:
            for s in list(self._solvers):  # a solver's buffers live on this context's stream
                s.close()
            load().lsg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        call("lsg_ctx_synchronize", self.h)

    def fp64_rate(self):
        """Measured FP64 DADD/DMUL issue rate of this device (instructions/s)."""
        r = C.c_double()
        call("lsg_probe_fp64_rate", self.h, C.byref(r))
        return r.value

    def comm_info(self):
        """(nranks, rank) as the NCCL communicator reports them; (0, -1) without one."""
        n, r = C.c_int(), C.c_int()
        call("lsg_ctx_comm_info", self.h, C.byref(n), C.byref(r))
        return n.value, r.value

    def local_nodes(self, g):
        """Nodes this process holds of grid g: the whole grid, or on a
        multi-rank context this rank's slab along the last axis (the size of
        the fields the solver-backed calls take and return)."""
        N = node_count(g)
        if self.nranks > 1:
            n = g.counts[g.dim - 1]
            _, nz = slab_partition(n, self.nranks, self.rank)
            N = N // n * nz
        return N

    def launches(self):
        n = C.c_uint64()
        call("lsg_ctx_launch_count", self.h, C.byref(n))
        return n.value

    # ---- stateless reference-facing calls --------------------------------
    def pad_ghost(self, g, v, dim, width):
        v = np.ascontiguousarray(v, dtype=np.float64)
        n = g.counts[dim] if 0 <= dim < g.dim else 1
        out = np.empty(max(1, node_count(g) // max(n, 1) * (n + 2 * max(width, 0))), dtype=np.float64)
        call("lsg_pad_ghost", self.h, C.byref(g), abi.dptr(v), C.c_int(dim), C.c_int(width), abi.dptr(out))
        return out

    def shift_along_dim(self, g, padded, dim, width, offset):
        padded = np.ascontiguousarray(padded, dtype=np.float64)
        out = np.empty(node_count(g), dtype=np.float64)
        call("lsg_shift_along_dim", self.h, C.byref(g), abi.dptr(padded), C.c_int(dim), C.c_int(width),
             C.c_int(offset), abi.dptr(out))
        return out

    def upwind(self, g, v, dim, scheme):
        v = np.ascontiguousarray(v, dtype=np.float64)
        L = np.empty(node_count(g), dtype=np.float64)
        R = np.empty(node_count(g), dtype=np.float64)
        call("lsg_upwind", self.h, C.byref(g), abi.dptr(v), C.c_int(dim), C.c_int(scheme), abi.dptr(L),
             abi.dptr(R))
        return L, R

    def term_lf(self, g, p, t, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty(self.local_nodes(g), dtype=np.float64)
        if v.size != out.size:
            raise ValueError("term_lf: field size does not match the (local) node count")
        b = C.c_double()
        call("lsg_term_lf", self.h, C.byref(g), C.byref(p), C.c_double(t), abi.dptr(v), abi.dptr(out), C.byref(b))
        return out, b.value

    def eval_hamiltonian(self, g, p, costate, t=0.0):
        """The device Hamiltonian on host costate fields (HamiltonianFn)."""
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in costate]
        arr = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
        out = np.empty(node_count(g), dtype=np.float64)
        call("lsg_eval_hamiltonian", self.h, C.byref(g), C.byref(p), C.c_double(t), arr, abi.dptr(out))
        return out

    def eval_dissipation(self, g, p, dim, t=0.0):
        """The device dissipation bound of dimension dim (DissipationFn)."""
        out = np.empty(node_count(g), dtype=np.float64)
        call("lsg_eval_dissipation", self.h, C.byref(g), C.byref(p), C.c_double(t), C.c_int(dim), abi.dptr(out))
        return out

    def set_op(self, op, a, b=None):
        """set_union (1) / set_intersection (2) / set_complement (3) of host fields on the device."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = a if b is None else np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty_like(a)
        call("lsg_set_op", self.h, C.c_int(op), C.c_size_t(a.size), abi.dptr(a), abi.dptr(b), abi.dptr(out))
        return out

    def restrict_update(self, dvdt, direction):
        dvdt = np.ascontiguousarray(dvdt, dtype=np.float64)
        out = np.empty_like(dvdt)
        call("lsg_restrict_update", self.h, C.c_size_t(dvdt.size), abi.dptr(dvdt), C.c_int(direction),
             abi.dptr(out))
        return out

    def integrate(self, g, p, method, t0, tf, v0, opts=None, log_cap=4096):
        v = np.array(v0, dtype=np.float64, copy=True)
        n = C.c_size_t()
        tfin = C.c_double()
        while True:  # LSG_ERANGE reports the log size a leg needs before anything runs
            log = (abi.LsgStepLog * log_cap)()
            rc = load().lsg_integrate(self.h, C.byref(g), C.byref(p), C.c_int(method), C.c_double(t0),
                                      C.c_double(tf), abi.dptr(v), C.byref(opts) if opts is not None else None, log,
                                      C.c_size_t(log_cap), C.byref(n), C.byref(tfin))
            if rc == abi.ERANGE and n.value > log_cap:
                log_cap = n.value
                continue
            raise_for(rc)
            return v, _steps(log, n.value, log_cap), tfin.value

    def gather_field(self, g, local):
        """Global field on rank 0 from this rank's slab (lsg_gather_field;
        collective on a multi-rank context, None on the other ranks)."""
        local = np.ascontiguousarray(local, dtype=np.float64)
        root = self.nranks <= 1 or self.rank == 0
        out = np.empty(node_count(g), dtype=np.float64) if root else None
        call("lsg_gather_field", self.h, C.byref(g), abi.dptr(local), abi.dptr(out) if root else None)
        return out

    def solve_brt(self, g, p, v0, tspan, n_checkpoints, method=abi.CFL3, opts=None, log_cap=4096, gather=False):
        """solve_brt (reachability.cpp:135-174).  On a multi-rank context v0 and
        the checkpoints are this rank's slab; gather=True returns whole-grid
        checkpoints on rank 0 instead (None on the other ranks)."""
        v0 = np.ascontiguousarray(v0, dtype=np.float64)
        N = self.local_nodes(g)
        if v0.size != N:
            raise ValueError("solve_brt: field size does not match the (local) node count")
        ck = np.empty(max(1, n_checkpoints) * N, dtype=np.float64)
        times = np.empty(max(1, n_checkpoints), dtype=np.float64)
        n_out = C.c_int()
        n = C.c_size_t()
        secs = C.c_double()
        while True:
            log = (abi.LsgStepLog * log_cap)()
            rc = load().lsg_solve_brt(self.h, C.byref(g), C.byref(p), abi.dptr(v0), C.c_double(tspan[0]),
                                      C.c_double(tspan[1]), C.c_int(n_checkpoints), C.c_int(method),
                                      C.byref(opts) if opts is not None else None, abi.dptr(ck), abi.dptr(times),
                                      C.byref(n_out), log, C.c_size_t(log_cap), C.byref(n), C.byref(secs))
            if rc == abi.ERANGE and n.value > log_cap:
                log_cap = n.value
                continue
            raise_for(rc)
            break
        k = n_out.value
        ck = ck[: k * N].reshape(k, N)
        if gather and self.nranks > 1:
            full = [self.gather_field(g, ck[j]) for j in range(k)]
            ck = np.stack(full) if self.rank == 0 else None
        return ck, times[:k].copy(), _steps(log, n.value, log_cap), secs.value


    def solve_brt_resume(self, g, p, v_k, k, t_k, tspan, n_checkpoints, method=abi.CFL3, opts=None, log_cap=4096):
        """Continue a solve_brt from checkpoint k (field v_k at integration time
        t_k): the checkpoints k .. n-1, their times, the remaining step log."""
        v_k = np.ascontiguousarray(v_k, dtype=np.float64)
        N = self.local_nodes(g)
        if v_k.size != N:
            raise ValueError("solve_brt_resume: field size does not match the (local) node count")
        m = max(1, n_checkpoints - k)
        ck = np.empty(m * N, dtype=np.float64)
        times = np.empty(m, dtype=np.float64)
        n_out, n, secs = C.c_int(), C.c_size_t(), C.c_double()
        while True:
            log = (abi.LsgStepLog * log_cap)()
            rc = load().lsg_solve_brt_resume(self.h, C.byref(g), C.byref(p), abi.dptr(v_k), C.c_int(k),
                                             C.c_double(t_k), C.c_double(tspan[0]), C.c_double(tspan[1]),
                                             C.c_int(n_checkpoints), C.c_int(method),
                                             C.byref(opts) if opts is not None else None, abi.dptr(ck),
                                             abi.dptr(times), C.byref(n_out), log, C.c_size_t(log_cap), C.byref(n),
                                             C.byref(secs))
            if rc == abi.ERANGE and n.value > log_cap:
                log_cap = n.value
                continue
            raise_for(rc)
            break
        j = n_out.value
        return ck[: j * N].reshape(j, N), times[:j].copy(), _steps(log, n.value, log_cap), secs.value

    def extract_zero_set_2d(self, g, field):
        """Marching-squares zero contour (contour.cpp:27-97): array (n, 4) of ax, ay, bx, by."""
        field = np.ascontiguousarray(field, dtype=np.float64)
        n = C.c_size_t()
        cap = 4096
        while True:
            seg = np.empty((cap, 4), dtype=np.float64)
            rc = load().lsg_extract_zero_set_2d(self.h, C.byref(g), abi.dptr(field), abi.dptr(seg), C.c_size_t(cap),
                                                C.byref(n))
            if rc == abi.ERANGE and n.value > cap:
                cap = n.value
                continue
            raise_for(rc)
            return seg[: n.value].copy()

    def slice_2d(self, g, field, fixed_dim, index):
        """contour.cpp:99-135: the 2-D slice fixed_dim = index of a 3-D field."""
        field = np.ascontiguousarray(field, dtype=np.float64)
        kept = [d for d in range(g.dim) if d != fixed_dim]
        out = np.empty(g.counts[kept[0]] * g.counts[kept[1]] if len(kept) == 2 else 1, dtype=np.float64)
        call("lsg_slice_2d", self.h, C.byref(g), abi.dptr(field), C.c_int(fixed_dim), C.c_int(index), abi.dptr(out))
        return out


class Solver:
    """Device-resident value function (lsg_solver): the fast path."""

    def __init__(self, ctx: Context, g, p, method, nslabs=1):
        self.h = None
        self.ctx = ctx
        self.g, self.p, self.method = g, p, method
        h = C.c_void_p()
        if nslabs == 1:
            call("lsg_solver_create", ctx.h, C.byref(g), C.byref(p), C.c_int(method), C.byref(h))
        else:
            call("lsg_solver_create_slabs", ctx.h, C.byref(g), C.byref(p), C.c_int(method), C.c_int(nslabs),
                 C.byref(h))
        self.h = h
        z0, nz, nodes = C.c_int(), C.c_int(), C.c_size_t()
        call("lsg_solver_slab", h, C.byref(z0), C.byref(nz), C.byref(nodes))
        self.z0, self.nz, self.local_nodes = z0.value, nz.value, nodes.value
        ctx._solvers.add(self)

    def close(self):
        if self.h:
            if self.ctx.h:  # a closed context already released its solvers
                load().lsg_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_field(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.size != self.local_nodes:
            raise ValueError("field: data size does not match the local node count")
        call("lsg_solver_set_field", self.h, abi.dptr(v))

    def get_field(self, out=None):
        """Download the resident field (into `out`, e.g. a pinned buffer, when given)."""
        if out is None:
            out = np.empty(self.local_nodes, dtype=np.float64)
        elif out.dtype != np.float64 or out.size != self.local_nodes or not out.flags.c_contiguous:
            raise ValueError("get_field: out must be a contiguous float64 array of local_nodes values")
        call("lsg_solver_get_field", self.h, abi.dptr(out))
        return out

    def set_field_device(self, ptr):
        call("lsg_solver_set_field_device", self.h, C.c_void_p(ptr))

    def field_device(self):
        p = C.c_void_p()
        call("lsg_solver_field_device", self.h, C.byref(p))
        return p.value

    def init_shape(self, shape, center, radius, ignored_dims=()):
        mask = 0
        for d in ignored_dims:
            mask |= 1 << d
        c = np.zeros(abi.MAX_DIM, dtype=np.float64)
        c[: len(center)] = center
        call("lsg_solver_init_shape", self.h, C.c_int(shape), C.c_uint(mask), abi.dptr(c), C.c_double(radius))

    def apply_shape(self, op, shape, center=None, radius=1.0, ignored_dims=(), upper=None):
        """Compose an implicit surface into the resident field on the device
        (lsg_solver_apply_shape): op 0 replace, 1 union, 2 intersection; shape
        0 sphere, 1 cylinder, 2 pair distance, 3 rectangle (center = lower
        corner, upper), 4 ellipsoid (radius)."""
        D = self.g.dim
        c = (C.c_double * 6)(*(list(center) if center is not None else [0.0] * D))
        u = (C.c_double * 6)(*(list(upper) if upper is not None else [0.0] * D))
        mask = 0
        for d in ignored_dims:
            mask |= 1 << d
        call("lsg_solver_apply_shape", self.h, C.c_int(op), C.c_int(shape), C.c_uint(mask), c, u,
             C.c_double(radius))

    def complement(self):
        call("lsg_solver_complement", self.h)

    def step_bound(self, t=0.0):
        b = C.c_double()
        call("lsg_solver_step_bound", self.h, C.c_double(t), C.byref(b))
        return b.value

    def step(self, t, dt):
        call("lsg_solver_step", self.h, C.c_double(t), C.c_double(dt))

    def step_host(self, t, dt, v, out=None):
        """One step from a host field to a host result, copies overlapped with
        the kernels (lsg_solver_step_host).  `out` may be `v` (in place)."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.size != self.local_nodes:
            raise ValueError("step_host: field size does not match the solver's local node count")
        if out is None:
            out = np.empty(self.local_nodes, dtype=np.float64)
        elif out.dtype != np.float64 or out.size != self.local_nodes or not out.flags.c_contiguous:
            raise ValueError("step_host: out must be a contiguous float64 array of local_nodes values")
        call("lsg_solver_step_host", self.h, C.c_double(t), C.c_double(dt), abi.dptr(v), abi.dptr(out))
        return out

    def step_timed(self, t, dt):
        """One step with device timing: (per-stage ms list, whole-step ms)."""
        stage = (C.c_double * 8)()
        total = C.c_double()
        call("lsg_solver_step_timed", self.h, C.c_double(t), C.c_double(dt), stage, C.byref(total))
        return [stage[k] for k in range(self.method + 1)], total.value

    def integrate(self, t0, tf, opts=None, log_cap=4096):
        n = C.c_size_t()
        tfin = C.c_double()
        while True:
            log = (abi.LsgStepLog * log_cap)()
            rc = load().lsg_solver_integrate(self.h, C.c_double(t0), C.c_double(tf),
                                             C.byref(opts) if opts is not None else None, log, C.c_size_t(log_cap),
                                             C.byref(n), C.byref(tfin))
            if rc == abi.ERANGE and n.value > log_cap:
                log_cap = n.value
                continue
            raise_for(rc)
            return _steps(log, n.value, log_cap), tfin.value

    def write_snapshot(self, time, path):
        """Reference-format snapshot of the resident field; collective on a
        multi-rank context (rank 0 writes the whole grid)."""
        call("lsg_solver_write_snapshot", self.h, C.c_double(time), str(path).encode() if path is not None else None)

    def stream(self):
        p = C.c_void_p()
        call("lsg_solver_stream", self.h, C.byref(p))
        return p.value

    def launches_per_step(self):
        n = C.c_int()
        call("lsg_solver_launches_per_step", self.h, C.byref(n))
        return n.value


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    call("lsg_nccl_unique_id", buf)
    return bytes(buf)


class PinnedArray:
    """float64 numpy view of a page-locked buffer from lsg_host_alloc.
    Keep this object alive while `array` is in use (freeing it unpins the memory)."""

    def __init__(self, n):
        p = C.c_void_p()
        call("lsg_host_alloc", C.c_size_t(8 * max(1, n)), C.byref(p))
        self.ptr = p
        self.array = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=(n,))

    def free(self):
        if self.ptr:
            self.array = None
            load().lsg_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def write_snapshot(g, field, time, path):
    """snapshot.cpp:69-93 format (host-only)."""
    field = np.ascontiguousarray(field, dtype=np.float64)
    call("lsg_write_snapshot", C.byref(g), abi.dptr(field), C.c_double(time), str(path).encode())


def read_snapshot(path):
    """(grid, field, time) from a snapshot.cpp:95-129 file (host-only)."""
    g = abi.LsgGrid()
    t = C.c_double()
    call("lsg_read_snapshot", str(path).encode(), C.byref(g), C.byref(t), None, C.c_size_t(0))
    out = np.empty(node_count(g), dtype=np.float64)
    call("lsg_read_snapshot", str(path).encode(), C.byref(g), C.byref(t), abi.dptr(out), C.c_size_t(out.size))
    return g, out, t.value


def slab_partition(n, nranks, rank):
    """(z0, nz) of rank's slab along an axis of n planes (host-only)."""
    z0, nz = C.c_int(), C.c_int()
    call("lsg_slab_partition", C.c_int(n), C.c_int(nranks), C.c_int(rank), C.byref(z0), C.byref(nz))
    return z0.value, nz.value


def halo_plan(n, nranks, rank, width, periodic):
    """The halo messages of rank's exchange in issue order (lsg_halo_plan,
    host-only): list of (kind 'send'|'recv', peer, first plane, planes)."""
    k, p, pl, c = (C.c_int * 4)(), (C.c_int * 4)(), (C.c_int * 4)(), (C.c_int * 4)()
    m = C.c_int()
    call("lsg_halo_plan", C.c_int(n), C.c_int(nranks), C.c_int(rank), C.c_int(width), C.c_int(1 if periodic else 0),
         k, p, pl, c, C.byref(m))
    return [("send" if k[i] == 0 else "recv", p[i], pl[i], c[i]) for i in range(m.value)]


def device_count():
    n = C.c_int()
    call("lsg_device_count", C.byref(n))
    return n.value
