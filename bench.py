#!/usr/bin/env python3
"""bench.py — grid-point updates/s per RK stage of the fused HJ hot path on B200.

Default workload (N=1): BASELINE.json configs[4], the largest single-GPU
configuration — 3-D motion in the normal direction on a 512^3 periodic grid
(134,217,728 nodes, 1.07 GB per field), WENO5 Lax-Friedrichs + TVD-RK3, fp64,
synthetic sphere initial level set built on the device.  `value` is the
bit-exact WENO5 path; ENO3 and the 1e-10-tolerance WENO5 ("weno5-fast") on
the same grid are printed under `extras`, each with its own HBM and FP64
roofline fractions.  One "step" = one RK3 step = 3 fused stage kernels.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config cfg5|cfg4|cfg3|cfg2] [--scheme weno5|weno5-fast|eno3|eno2|first]

* value   device-resident (inputs in HBM), one CUDA event pair on the
          launching stream around the K timed steps, max over ranks;
          pt-stage/s = nodes * 3 * K / time.  Fields are 8x the 126 MB L2, so
          no flush is needed between steps (cfg2's 8 MB fields are flushed).
* e2e     the same metric through the public C ABI with host buffers: every
          step copies the value function in from pinned host memory and the
          result back (lsg_solver_step_host; copies overlapped with compute).
* roofline  the dominant kernel (the COMBINE stage, 24 algorithmic B/node):
          its average launch time is the timed step time times its share of
          the step (per-stage events of untimed steps), DRAM traffic from the
          committed ncu capture of this command (profiles/), HBM peak from
          MEASURED_PEAKS.json; roofline_fp64 against the FP64 issue rate
          measured in this run (lsg_probe_fp64_rate).
* --gpus N  without torchrun: spawns N ranks with torch.distributed.run
          (127.0.0.1).  cfg5 is weak scaling (512 x 512 x 512*N, slabs along
          z, NCCL halo send/recv); cfg4 (41^6) and cfg3 are strong scaling.
* --impl reference  the reference's own CPU implementation (oracle/_ref,
          compiled from /root/reference sources) on the host's cores: R
          concurrent replicas of integrate() on a stated bounded sample of the
          same workload, R = min(host threads, RAM / replica footprint).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2507_11542_b200 import abi  # noqa: E402
from paper_2507_11542_b200 import problems as P  # noqa: E402

METRIC = "grid-point updates/sec per RK stage (ENO3/WENO5 LF); HBM GB/s vs peak"
UNIT = "pt-stage/s"
# compulsory HBM bytes per point of a fused stage: stage 1 reads v
# and writes v1 (16 B); stages 2 and 3 read two fields and write one (24 B).
BYTES_EULER, BYTES_COMBINE = 16.0, 24.0
BYTES_PER_PT_STAGE = {abi.CFL1: 16.0, abi.CFL2: 20.0, abi.CFL3: 64.0 / 3.0}
L2_BYTES = 126 * 1024 * 1024

SCHEMES = {  # name -> (scheme id, options, label)
    "first": (abi.SCHEME_FIRST, 0, "First"),
    "eno2": (abi.SCHEME_ENO2, 0, "ENO2"),
    "eno3": (abi.SCHEME_ENO3, 0, "ENO3"),
    "weno5": (abi.SCHEME_WENO5, 0, "WENO5 (bit-exact)"),
    "weno5-fast": (abi.SCHEME_WENO5, abi.OPT_WENO5_FAST, "WENO5 fast (1e-10 tolerance)"),
}
DEFAULT_SCHEME = {"cfg5": "weno5", "cfg4": "weno5", "cfg3": "weno5", "cfg2": "eno3"}


# ---------------------------------------------------------------------------
# workloads

def workload(cfg, scheme, ws):
    """(Setup, config dict, scaling) of the run; the config dict is identical
    in both arms (the reference arm samples it, see cpu_sample)."""
    sid, opt, label = SCHEMES[scheme]
    if cfg == "cfg5":
        S = P.cfg5_normal(512, sid, z_scale=ws)
        name = "cfg5_normal_512^3_%s_lf_rk3" % scheme if ws == 1 else "cfg5_normal_512x512x%d_%s_lf_rk3_weak" % (
            512 * ws, scheme)
        scaling = "weak"
    elif cfg == "cfg4":
        S = P.cfg4_dubins6(41, sid)
        name = "cfg4_dubins6_41^6_%s_lf_rk3" % scheme
        scaling = "strong"
    elif cfg == "cfg3":
        S = P.cfg3_dblint4(81)
        S.problem.scheme = sid
        name = "cfg3_dblint4_81^4_%s_lf_rk3" % scheme
        scaling = "strong"
    elif cfg == "cfg2":
        S = P.cfg2_air3d(101, z_scale=ws)
        S.problem.scheme = sid
        name = "cfg2_air3d_101^3_%s_lf_rk3" % scheme if ws == 1 else "cfg2_air3d_101x101x%d_%s_lf_rk3_weak" % (
            101 * ws, scheme)
        scaling = "weak"
    else:
        raise SystemExit(f"unknown --config {cfg}")
    S.problem.options = opt
    grid = [S.grid.counts[d] for d in range(S.grid.dim)]
    nodes = 1
    for n in grid:
        nodes *= n
    field_bytes = 8 * nodes
    config = {
        "workload": name,
        "grid": grid,
        "nodes": nodes,
        "scheme": label,
        "hamiltonian": abi.HAM_NAMES[S.problem.kind],
        "integrator": {abi.CFL1: "odeCFL1", abi.CFL2: "odeCFL2", abi.CFL3: "odeCFL3 (TVD-RK3)"}[S.method],
        "clamp": ("Grow" if S.problem.direction == abi.GROW else "Shrink") if S.problem.restrict_update else "none",
        "parallelism": "single" if ws == 1 else f"slab{ws} (last axis, NCCL halo send/recv)",
        "l2": ("no flush: 3 fields of %.2f GB per GPU >> 126 MB L2" % (field_bytes / ws / 1e9))
        if field_bytes / ws > 4 * L2_BYTES else "flushed before every timed step (512 MiB write)",
    }
    return S, config, scaling


def cpu_sample(cfg, scheme):
    """Bounded sample of the workload for the reference's CPU path: a Setup
    whose per-node work matches the full grid's (same scheme, integrator,
    Hamiltonian, spacing and line lengths where possible) and a description."""
    sid, opt, _ = SCHEMES[scheme]
    if cfg == "cfg5":
        S = P.cfg5_normal(512, sid, nz=16)
        desc = "512x512x16 periodic slab of the cfg5 problem (same x/y lines, spacing and strides as 512^3)"
    elif cfg == "cfg4":
        S = P.cfg4_dubins6(13, sid)
        desc = "13^6 cfg4 Dubins grid (41^6 = 38 GB/field cannot run on the host)"
    elif cfg == "cfg3":
        S = P.cfg3_dblint4(41)
        S.problem.scheme = sid
        desc = "41^4 cfg3 double-integrator grid"
    else:
        S = P.cfg2_air3d(101)
        S.problem.scheme = sid
        desc = "full 101^3 cfg2 Air3D grid"
    S.problem.options = 0  # the reference has one WENO5
    return S, desc


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def avail_ram_bytes():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return 8 << 30


# the reference keeps ~20 full fields per integrate() call (v, RK buffers, D
# derivative pairs, D central fields, H, bounds, dvdt, D coordinate fields):
# 21.0 GB RSS measured at 512^3 WENO5 = 156 B/node
REF_BYTES_PER_NODE = 160


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback"


def ncu_capture(cfg, scheme):
    """Per-launch DRAM bytes and FP64 instructions per node of the dominant
    kernel from the committed ncu capture of this command (profiles/),
    keyed "<config>/<scheme>"."""
    path = os.path.join(ROOT, "profiles", "ncu_bench_captures.json")
    try:
        with open(path) as f:
            return json.load(f).get(f"{cfg}/{scheme}", {})
    except Exception:
        return {}


class ClockSampler:
    """SM clock + throttle reasons sampled by NVML during the timed region."""

    def __init__(self, device=0, period=0.02):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def spawn_ranks(n):
    """--gpus N outside torchrun: relaunch this command as N ranks."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    # communicator init (rank count, transports) goes to stderr, the JSON line to stdout
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------------------
# the reference's CPU path

def ref_run(S, replicas, steps, warmup=1, seconds_cap=90.0):
    """`replicas` concurrent reference integrate() calls of `steps` RK steps
    each on S (oracle/_ref, the reference compiled from its own sources)."""
    from oracle import oracle as O

    ref = O.reference()
    shape, center, radius, ignored = S.ic
    if shape == P.SPHERE:
        v0 = ref.sphere(S.grid, center, radius)
    elif shape == P.CYLINDER:
        v0 = ref.cylinder(S.grid, list(ignored), center, radius)
    else:  # cfg4's planar pair distance sqrt((xa-xb)^2 + (ya-yb)^2) - r (builder-defined)
        g = S.grid
        ax = [ref.axis(g, d) for d in range(g.dim)]
        mesh = np.meshgrid(*ax, indexing="ij")  # column-major flattening below
        a = (mesh[0] - mesh[3]).ravel(order="F")
        b = (mesh[1] - mesh[4]).ravel(order="F")
        v0 = np.sqrt((0.0 + a * a) + b * b) - radius
    _, bound = ref.term_lf(S.grid, S.problem, 0.0, v0)
    dt = 0.32 * bound
    opts = abi.make_opts(max_step=dt)
    ws_, wsteps = ref.bench(S.grid, S.problem, S.method, v0, max(1, warmup) * dt, opts, replicas)
    per_step = ws_ / max(wsteps, 1)
    k = max(1, min(steps, int(seconds_cap / max(per_step, 1e-9))))
    secs, nsteps = ref.bench(S.grid, S.problem, S.method, v0, k * dt, opts, replicas)
    nodes = v0.size
    return replicas * nodes * (S.method + 1) * nsteps / secs, nsteps, secs, nodes


def reference_arm(args):
    """--impl reference: the reference's own CPU implementation of the path."""
    ws, rank, _ = dist_env()
    n_gpus = max(ws, args.gpus)
    if rank != 0:
        return 0
    from oracle import oracle as O

    scheme = args.scheme or DEFAULT_SCHEME[args.config]
    _, config, scaling = workload(args.config, scheme, n_gpus)
    if not O.have_reference():
        print(json.dumps({"impl": "reference", "metric": METRIC,
                          "unavailable": "oracle/_ref/libref_levelset.so was not built"}))
        return 0
    S, desc = cpu_sample(args.config, scheme)
    nodes = 1
    for d in range(S.grid.dim):
        nodes *= S.grid.counts[d]
    threads = host_threads()
    ram = avail_ram_bytes()
    replicas = max(1, min(threads, int(0.7 * ram // (REF_BYTES_PER_NODE * nodes))))
    value, steps, secs, _ = ref_run(S, replicas, args.steps, args.warmup, seconds_cap=args.ref_seconds)
    sample = (f"{steps} RK{S.method + 1} steps of a {desc} ({nodes} nodes) in each of {replicas} concurrent "
              f"replica threads (replicas = min({threads} host threads, 0.7 x {ram / 2**30:.0f} GiB available / "
              f"{REF_BYTES_PER_NODE} B/node)); host: {threads} threads, {cpu_model()}")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": n_gpus,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / max(steps, 1),
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": replicas, "kind": "reference", "sample": sample,
                         "host_threads": threads, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "path": "oracle/_ref: the reference levelset core compiled from /root/reference sources; "
                "integrate(Cfl3, term_lax_friedrichs) per replica thread (bench_kernels.cpp:70-83 pattern)",
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# the B200 arm

class Timed:
    """K steps of a device-resident solver, one event pair around all of them
    (or around each step after an L2 flush), plus the stage shares."""

    def __init__(self, torch, ctx, solver, dt, stream, flush=None):
        self.torch, self.ctx, self.solver, self.dt, self.stream, self.flush = torch, ctx, solver, dt, stream, flush
        self.t = 0.0

    def warm(self, n):
        for _ in range(n):
            self.solver.step(self.t, self.dt)
            self.t += self.dt
        self.ctx.synchronize()

    def run(self, k, barrier):
        torch = self.torch
        launches0 = self.ctx.launches()
        barrier()
        if self.flush is None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            for _ in range(k):
                self.solver.step(self.t, self.dt)
                self.t += self.dt
            e1.record(self.stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        else:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
            for a, b in evs:
                with torch.cuda.stream(self.stream):
                    self.flush.zero_()
                a.record(self.stream)
                self.solver.step(self.t, self.dt)
                self.t += self.dt
                b.record(self.stream)
            torch.cuda.synchronize()
            ms = float(sum(a.elapsed_time(b) for a, b in evs))
        barrier()
        return ms, self.ctx.launches() - launches0

    def stage_shares(self, n=3):
        st = []
        for _ in range(n):
            if self.flush is not None:
                with self.torch.cuda.stream(self.stream):
                    self.flush.zero_()
            st.append(self.solver.step_timed(self.t, self.dt)[0])
            self.t += self.dt
        m = np.array(st).mean(axis=0)
        return [float(x) for x in m / m.sum()], [float(x) for x in m]


def roofline(ms_per_step, shares, nodes_local, method, peak, peak_kind, fp64_peak, cap):
    """Dominant kernel = the COMBINE stage (RK2/RK3), else the EULER stage."""
    if method == abi.CFL1:
        share, nbytes, kern = shares[0], BYTES_EULER * nodes_local, "EULER"
    else:
        share = sum(shares[1:]) / (len(shares) - 1)
        nbytes, kern = BYTES_COMBINE * nodes_local, "COMBINE"
    launch_ms = ms_per_step * share
    achieved = nbytes / (launch_ms * 1e-3) / 1e9
    fp64_node = cap.get("fp64_instr_per_node")
    r = {
        "bound": "hbm",
        "kernel": f"fused {kern} stage ({cap.get('kernel_symbol', 'march3_kernel')})",
        "achieved": achieved,
        "peak": peak,
        "unit": "GB/s",
        "frac": achieved / peak,
        "traffic": cap.get("dram_bytes_per_launch"),
        "peak_kind": peak_kind,
        "algorithmic_bytes_per_launch": nbytes,
        "avg_launch_ms": launch_ms,
        "launch_ms_source": "timed step time x the stage's share of per-stage events in untimed steps",
        "traffic_source": cap.get("capture"),
    }
    r64 = None
    if fp64_node:
        a64 = fp64_node * nodes_local / (launch_ms * 1e-3)
        r64 = {"bound": "fp64", "achieved": a64, "peak": fp64_peak, "unit": "FP64 instr/s", "frac": a64 / fp64_peak,
               "instr_per_node": fp64_node,
               "source": "instr/node: ncu SASS opcode count of this kernel (profiles/ncu_bench_captures.json); "
                         "peak: DADD/DMUL issue rate measured in this run (lsg_probe_fp64_rate)"}
    return r, r64


def b200_arm(args):
    import torch

    from paper_2507_11542_b200 import _lib

    ws, rank, local = dist_env()
    dist = None
    if ws > 1 or args.dist_selftest:
        import torch.distributed as dist

        if ws == 1:  # one-rank NCCL communicator through the multi-rank branch
            os.environ["LSG_DIST_SELFTEST"] = "1"
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        # NCCL prints its version banner on stdout at the first communicator
        # init; keep stdout for the JSON line (the banner and INFO lines go to stderr)
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(_lib.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, 0)
            ctx = _lib.Context(local, rank, ws, bytes(uid.cpu().numpy().tobytes()))
            torch.cuda.synchronize()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
        n_comm, r_comm = ctx.comm_info()
        print(f"bench: rank {rank}: lsg NCCL communicator with {n_comm} ranks (this rank {r_comm})", file=sys.stderr)
    else:
        torch.cuda.set_device(0)
        ctx = _lib.Context(0)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    scheme = args.scheme or DEFAULT_SCHEME[args.config]
    S, config, scaling = workload(args.config, scheme, ws)
    peak, peak_kind = peaks()
    fp64_peak = ctx.fp64_rate()

    def build(setup):
        sol = _lib.Solver(ctx, setup.grid, setup.problem, setup.method)
        shape, center, radius, ignored = setup.ic
        sol.init_shape(shape, center, radius, ignored)
        return sol

    solver = build(S)
    bound = solver.step_bound()
    dt = 0.32 * bound
    nodes_local = solver.local_nodes
    nodes_total = config["nodes"]
    stages = S.method + 1
    stream = torch.cuda.ExternalStream(solver.stream())
    flush = None
    if 8 * nodes_local <= 4 * L2_BYTES:
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # ---- timed region ----------------------------------------------------
    T = Timed(torch, ctx, solver, dt, stream, flush)
    T.warm(args.warmup)
    sampler = ClockSampler(local)
    with sampler:
        ms, launches = T.run(args.steps, barrier)
    ms = max_over_ranks(ms)
    value = nodes_total * stages * args.steps / (ms * 1e-3)
    ms_per_step = ms / args.steps
    shares, stage_ms = T.stage_shares()
    cap = ncu_capture(args.config, scheme)
    roof, roof64 = roofline(ms_per_step, shares, nodes_local, S.method, peak, peak_kind, fp64_peak, cap)

    # ---- e2e: public C ABI with pinned host buffers -------------------------
    e2e = None
    e2e_leg = None
    if not args.no_e2e and 8 * nodes_local <= 8 * 2**30:
        pinned = _lib.PinnedArray(nodes_local)  # page-locked by the library's own CUDA runtime
        host_np = pinned.array
        solver.get_field(out=host_np)
        e2e_steps = max(1, min(args.steps, 20))
        t = T.t
        for _ in range(2):  # warm the path (copy streams and events are created on first use)
            solver.step_host(t, dt, host_np, out=host_np)
            t += dt
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            # H2D of the step's input, the step, D2H of its result: one
            # lsg_solver_step_host call (bit-identical to set_field + step + get_field)
            solver.step_host(t, dt, host_np, out=host_np)
            t += dt
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": nodes_total * stages * e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": 8 * nodes_local, "d2h_bytes_per_step": 8 * nodes_local, "steps": e2e_steps,
               "path": "lsg_solver_step_host per step: the full field H2D from pinned memory and the full result "
                       "D2H (single slab: chunked along z and overlapped with the stage kernels)"}
        # the reference arm's usage pattern: one stateless integrate() call over K steps
        if ws == 1:
            import ctypes as C

            lib = _lib.load()
            nlog = args.steps + 8
            log = (abi.LsgStepLog * nlog)()
            nst, tfin = C.c_size_t(), C.c_double()
            opts = abi.make_opts(max_step=dt)
            solver.close()  # the stateless call builds its own cached solver
            leg = lambda: lib.lsg_integrate(ctx.h, C.byref(S.grid), C.byref(S.problem), C.c_int(S.method),  # noqa
                                            C.c_double(0.0), C.c_double(args.steps * dt), pinned.ptr, C.byref(opts),
                                            log, C.c_size_t(nlog), C.byref(nst), C.byref(tfin))
            _lib.raise_for(leg())  # warm (builds the cached solver)
            t0 = time.perf_counter()
            _lib.raise_for(leg())
            leg_s = time.perf_counter() - t0
            e2e_leg = {"value": nodes_total * stages * nst.value / leg_s, "unit": UNIT, "steps": nst.value,
                       "h2d_bytes_per_call": 8 * nodes_local, "d2h_bytes_per_call": 8 * nodes_local,
                       "path": "one lsg_integrate call (the reference's integrate(term, {0, K*dt}, v0, {max_step}) "
                               "usage): pinned host field in, K steps, host field out"}
        pinned.free()
    solver.close()

    # ---- extras (N=1, cfg5): the other schemes on the same grid ---------------
    extras = {}
    if ws == 1 and args.config == "cfg5" and not args.no_extras:
        for name in ("eno3", "weno5-fast", "weno5"):
            if name == scheme:
                continue
            S2, c2, _ = workload("cfg5", name, 1)
            sol = build(S2)
            dt2 = 0.32 * sol.step_bound()
            T2 = Timed(torch, ctx, sol, dt2, stream, None)
            T2.warm(2)
            k2 = max(3, min(args.steps, 20))
            ms2, _ = T2.run(k2, barrier)
            sh2, _ = T2.stage_shares()
            r2, r64 = roofline(ms2 / k2, sh2, sol.local_nodes, S2.method, peak, peak_kind, fp64_peak,
                               ncu_capture("cfg5", name))
            extras[name] = {"workload": c2["workload"], "value": c2["nodes"] * 3 * k2 / (ms2 * 1e-3), "unit": UNIT,
                            "steps": k2, "ms_per_step": ms2 / k2,
                            "step_hbm_gbs": BYTES_PER_PT_STAGE[S2.method] * c2["nodes"] * 3 * k2 / (ms2 * 1e-3) / 1e9,
                            "roofline_frac_hbm": r2["frac"], "roofline_frac_fp64": r64["frac"] if r64 else None,
                            "fp64_instr_per_node": r64["instr_per_node"] if r64 else None,
                            "dram_bytes_per_launch": r2["traffic"]}
            sol.close()

    # ---- in-run scaling reference (N>1, weak scaling): the 1-GPU workload on rank 0
    eff = None
    if dist is not None and scaling == "weak" and not args.no_efficiency:  # (also under --dist-selftest)
        if rank == 0:
            # a plain single-GPU context: the distributed one would make the
            # solver collective (and wait for the idle ranks)
            ctx1 = _lib.Context(local)
            S1, c1, _ = workload(args.config, scheme, 1)
            sol = _lib.Solver(ctx1, S1.grid, S1.problem, S1.method)
            shape, center, radius, ignored = S1.ic
            sol.init_shape(shape, center, radius, ignored)
            stream1 = torch.cuda.ExternalStream(sol.stream())
            T1 = Timed(torch, ctx1, sol, 0.32 * sol.step_bound(), stream1, flush)
            T1.warm(args.warmup)
            ms1, _ = T1.run(args.steps, lambda: torch.cuda.synchronize())
            v1 = c1["nodes"] * stages * args.steps / (ms1 * 1e-3)
            eff = {"value_1gpu_same_run": v1, "weak_scaling_efficiency": value / (ws * v1),
                   "note": "rank 0 re-runs the N=1 workload on a single-GPU context after the timed multi-rank "
                           "region (other ranks idle); the driver's own SCALE efficiency uses the separate N=1 run"}
            sol.close()
            ctx1.close()
        if dist is not None:
            dist.barrier()

    nccl = None
    if dist is not None:
        n, r = ctx.comm_info()
        nccl = {"comm_nranks": n, "comm_rank": r, "backend": "NCCL (lsg ctx communicator) + torch.distributed"}

    if rank != 0:
        ctx.close()
        dist.destroy_process_group()
        return 0

    # ---- cpu_baseline: the reference on a bounded sample, 1 thread ------------
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O

        if O.have_reference():
            S3, desc = cpu_sample(args.config, scheme)
            v, steps, secs, nodes = ref_run(S3, 1, 1000, 0, seconds_cap=args.cpu_seconds)
            cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"{steps} RK{S3.method + 1} steps of a {desc} ({nodes} nodes), 1 thread, "
                             f"{secs:.1f} s (the reference is single-threaded); host {cpu_model()}, "
                             f"{host_threads()} threads"}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": config,
        "timing": {"timed_region_s": ms * 1e-3, "stage_ms_untimed": stage_ms, "stage_share": shares,
                   "alpha_dt": [bound, dt], "nodes_per_gpu": nodes_local,
                   "method": "one CUDA event pair on the launching stream around the K steps (per step after an "
                             "L2 flush when the fields fit L2); max over ranks"},
        "gpu_launches": launches,
        "roofline": roof,
        "roofline_fp64": roof64,
        "step_hbm_gbs": BYTES_PER_PT_STAGE[S.method] * value / 1e9,
        "e2e": e2e,
        "e2e_leg": e2e_leg,
        "clocks": sampler.summary(),
    }
    if e2e is None and not args.no_e2e:
        line["e2e_note"] = (f"not measured: the per-step host round trip of a {8 * nodes_local / 1e9:.1f} GB field "
                            "needs that much pinned host memory twice over (measured up to 8 GiB fields)")
    if extras:
        line["extras"] = extras
    if eff:
        line["efficiency"] = eff
    if nccl:
        line["nccl"] = nccl
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg5", choices=["cfg5", "cfg4", "cfg3", "cfg2"])
    ap.add_argument("--scheme", default=None, choices=sorted(SCHEMES))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-efficiency", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=90.0)
    ap.add_argument("--dist-selftest", action="store_true",
                    help="under torchrun with one rank: run the multi-rank (NCCL) branch on a one-rank communicator")
    ap.add_argument("--launch-check", action="store_true",
                    help="each rank prints its rank / world size and exits (tests the --gpus N launcher on CPU)")
    args = ap.parse_args()
    if args.launch_check and "WORLD_SIZE" in os.environ:
        ws, rank, local = dist_env()
        print(json.dumps({"launch_check": True, "rank": rank, "world_size": ws, "local_rank": local,
                          "master_addr": os.environ.get("MASTER_ADDR"), "nccl_debug": os.environ.get("NCCL_DEBUG")}),
              flush=True)
        return 0
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "b200" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return reference_arm(args)
    return b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
