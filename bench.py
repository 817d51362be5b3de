#!/usr/bin/env python3
"""bench.py — grid-point updates/s per RK stage of the fused HJ hot path on B200.

Workload (BASELINE.json configs[1], the config the metric is quoted on):
Air3D pursuit-evasion BRT, 101^3 grid, ENO3 Lax-Friedrichs + TVD-RK3, fp64,
heading axis periodic, Grow clamp, synthetic initial level set (cylinder of
radius 5, built on the device).  One "step" = one RK3 step = 3 fused stage
kernels over all 1,030,301 nodes (+ the fused v-range reduction).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

* value   device-resident (inputs in HBM), CUDA events around each step on the
          launching stream, L2 flushed (512 MiB write) before every timed step;
          pt-stage/s = nodes * 3 * K / sum(step times), max over ranks.
* e2e     the same metric through the public C ABI with host buffers: every
          step copies the value function in from pinned host memory
          (lsg_solver_set_field), runs the step, and copies it back
          (lsg_solver_get_field).
* --impl reference   the reference's own CPU implementation (oracle/_ref,
          compiled from /root/reference sources) on the host's cores: one
          replica per host thread, each a full 101^3 RK3 step per bench step.

Multi-GPU (torchrun): weak scaling, each rank holds a 101x101x101 slab of a
101x101x(101*N) Air3D grid (heading axis refined N times, periodic ring);
ghost planes move by NCCL send/recv between stages.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
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
BYTES_STAGE = {0: 16.0, 1: 24.0, 2: 24.0}
BYTES_PER_PT_STAGE_RK3 = 64.0 / 3.0


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


def ncu_summary():
    """Per-launch numbers of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# FP64 DADD/DMUL issue rate of one B200 (tools/fp64_peak.cu, measured under gpurun):
# 18.5 T instructions/s = 64 per SM per clock at 1.965 GHz.
FP64_PEAK = 18.5e12


def cpu_reference_sample(setup, v0, seconds_target=10.0, nthreads=1):
    """The reference CPU path (oracle/_ref) on a bounded sample of the workload:
    whole RK3 steps of the same 101^3 problem, `nthreads` replicas."""
    from oracle import oracle as O

    if not O.have_reference():
        return None, None
    ref = O.reference()
    N = v0.size
    _, bound = ref.term_lf(setup.grid, setup.problem, 0.0, v0)
    dt = 0.32 * bound
    secs1, steps1 = ref.bench(setup.grid, setup.problem, setup.method, v0, dt, abi.make_opts(max_step=dt), nthreads)
    k = max(1, int(seconds_target / max(secs1, 1e-6)))
    secs, steps = ref.bench(setup.grid, setup.problem, setup.method, v0, k * dt, abi.make_opts(max_step=dt),
                            nthreads)
    value = nthreads * N * 3 * steps / secs
    return value, {"steps": steps, "seconds": secs, "replicas": nthreads}


def reference_arm(args):
    """--impl reference: the reference's own CPU implementation of the path."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O

    setup = P.cfg2_air3d(101)
    if not O.have_reference():
        print(json.dumps({"impl": "reference", "metric": METRIC,
                          "unavailable": "oracle/_ref/libref_levelset.so was not built"}))
        return 0
    ref = O.reference()
    v0 = ref.cylinder(setup.grid, [2], [0.0, 0.0, 0.0], 5.0)
    N = v0.size
    _, bound = ref.term_lf(setup.grid, setup.problem, 0.0, v0)
    dt = 0.32 * bound
    try:
        threads = len(os.sched_getaffinity(0))
    except Exception:
        threads = os.cpu_count() or 1
    opts = abi.make_opts(max_step=dt)
    # warm-up (>= 1 step) doubles as the probe that bounds the sample to ~90 s
    w = max(1, args.warmup)
    wsecs, wsteps = ref.bench(setup.grid, setup.problem, setup.method, v0, w * dt, opts, threads)
    per_step = wsecs / max(wsteps, 1)
    k = max(1, min(args.steps, int(90.0 / max(per_step, 1e-9))))
    secs, steps = ref.bench(setup.grid, setup.problem, setup.method, v0, k * dt, opts, threads)
    value = threads * N * 3 * steps / secs
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / max(steps, 1),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "cfg2_air3d_101^3_eno3_lf_rk3", "nodes": N, "replicas": threads,
                   "path": "oracle/_ref: reference levelset core compiled from /root/reference sources, "
                           "integrate(Cfl3, term_lax_friedrichs) per replica thread"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{steps} RK3 steps of the full 101^3 Air3D problem in each of {threads} "
                                   f"concurrent replica threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def b200_arm(args):
    import torch

    from paper_2507_11542_b200 import _lib

    ws, rank, local = dist_env()
    dist = None
    if ws > 1 or args.dist_selftest:
        import torch.distributed as dist

        if ws == 1:  # one-rank NCCL communicator through the multi-rank branch
            os.environ["LSG_DIST_SELFTEST"] = "1"
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(_lib.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        ctx = _lib.Context(local, rank, ws, bytes(uid.cpu().numpy().tobytes()))
    else:
        torch.cuda.set_device(0)
        ctx = _lib.Context(0)

    setup = P.cfg2_air3d(101, z_scale=ws)
    solver = _lib.Solver(ctx, setup.grid, setup.problem, setup.method)
    shape, center, radius, ignored = setup.ic
    solver.init_shape(shape, center, radius, ignored)
    bound = solver.step_bound()
    dt = 0.32 * bound
    nodes_local = solver.local_nodes
    nodes_total = _lib.node_count(setup.grid)
    stages = setup.method + 1

    stream = torch.cuda.ExternalStream(solver.stream())
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up --------------------------------------------------------
    t = 0.0
    for _ in range(args.warmup):
        solver.step(t, dt)
        t += dt
    ctx.synchronize()

    # ---- timed region: K steps, L2 flushed before each -------------------
    # Each step is bracketed by one event pair on the launching stream (no
    # events between its stages, so consecutive stage kernels overlap their
    # launch ramp through programmatic dependent launch).
    launches0 = ctx.launches()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    barrier()
    with sampler:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                evs[k][0].record(stream)
            solver.step(t, dt)
            with torch.cuda.stream(stream):
                evs[k][1].record(stream)
            t += dt
        torch.cuda.synchronize()
    barrier()
    launches = ctx.launches() - launches0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    sum_ms = float(sum(step_ms))
    # per-stage breakdown for the roofline: separate, untimed steps with an
    # event after every stage (L2 flushed before each, like the timed steps)
    stage_ms = []
    for _ in range(20):
        with torch.cuda.stream(stream):
            flush.zero_()
        stage_ms.append(solver.step_timed(t, dt)[0])
        t += dt
    if dist is not None:
        tt = torch.tensor([sum_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        sum_ms = float(tt.item())
    value = nodes_total * stages * args.steps / (sum_ms * 1e-3)

    # dominant kernel: the fused COMBINE stage (stages 2 and 3, 24 B/pt algorithmic)
    st = np.array(stage_ms)
    comb_ms = float(st[:, 1:].mean()) if stages > 1 else float(st[:, 0].mean())
    comb_bytes = BYTES_STAGE[1] * nodes_local
    peak, peak_kind = peaks()
    achieved = comb_bytes / (comb_ms * 1e-3) / 1e9
    prof = ncu_summary()
    traffic = prof.get("dram_bytes_per_launch")

    # ---- e2e: public C ABI with pinned host buffers ------------------------
    pinned = _lib.PinnedArray(nodes_local)  # page-locked by the library's own CUDA runtime
    host_np = pinned.array
    solver.get_field(out=host_np)
    e2e_steps = max(1, min(args.steps, 200))
    for _ in range(max(1, args.warmup)):  # warm the path (copy streams and events are created on first use)
        solver.step_host(t, dt, host_np, out=host_np)
        t += dt
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(e2e_steps):
        # H2D of the step's input, the step, D2H of its result: one
        # lsg_solver_step_host call (copies chunked and overlapped with the
        # stage kernels; bit-identical to set_field + step + get_field)
        solver.step_host(t, dt, host_np, out=host_np)
        t += dt
    ev1.record(stream)
    barrier()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_value = nodes_total * stages * e2e_steps / e2e_s

    # ---- e2e_leg: the reference's usage pattern, one stateless integrate()
    # call over K steps (lsg_integrate: host field in, K steps, host field out)
    import ctypes as C
    lib = _lib.load()
    nlog = e2e_steps + 8
    log = (abi.LsgStepLog * nlog)()
    nst, tfin = C.c_size_t(), C.c_double()
    opts = abi.make_opts(max_step=dt)
    leg = lambda: lib.lsg_integrate(ctx.h, C.byref(setup.grid), C.byref(setup.problem), C.c_int(setup.method),
                                    C.c_double(0.0), C.c_double(e2e_steps * dt), pinned.ptr, C.byref(opts), log,
                                    C.c_size_t(nlog), C.byref(nst), C.byref(tfin))
    _lib.raise_for(leg())  # warm (builds the cached solver)
    barrier()
    t0 = time.perf_counter()
    _lib.raise_for(leg())
    barrier()
    leg_s = time.perf_counter() - t0
    if dist is not None:
        tt = torch.tensor([leg_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        leg_s = float(tt.item())
    leg_value = nodes_total * stages * nst.value / leg_s

    if rank != 0:
        dist.destroy_process_group()
        return 0

    cpu_value, cpu_info = (None, None)
    if ws == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O

        if O.have_reference():
            v0 = O.reference().cylinder(setup.grid, [2], [0.0, 0.0, 0.0], 5.0)
            cpu_value, cpu_info = cpu_reference_sample(setup, v0, seconds_target=args.cpu_seconds)

    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": sum_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": "cfg2_air3d_101^3_eno3_lf_rk3" if ws == 1 else f"cfg2_air3d_101x101x{101 * ws}_slabs",
            "grid": [setup.grid.counts[d] for d in range(setup.grid.dim)],
            "nodes_per_gpu": nodes_local,
            "scheme": "ENO3", "integrator": "odeCFL3 (TVD-RK3)", "clamp": "Grow",
            "parallelism": f"slab{ws}" if ws > 1 else ("slab1 (NCCL self-test)" if args.dist_selftest else "single"),
            "l2": "flushed before every timed step (512 MiB write); inputs 8.2 MB/field fit in L2",
            "timing": "one CUDA event pair on the launching stream around each step (after its L2 flush), "
                      "summed; max over ranks; per-stage times from 20 extra untimed steps",
            "stage_ms_mean": [float(x) for x in st.mean(axis=0)],
            "alpha_dt": [bound, dt],
        },
        "gpu_launches": launches,
        "roofline": {
            "bound": "hbm",
            "kernel": "march3_kernel<ENO3,AIR3D,COMBINE> (2.5-D tiled fused stage)",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": traffic,
            "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": comb_bytes,
            "avg_launch_ms": comb_ms,
            "step_gbs": BYTES_PER_PT_STAGE_RK3 * value / 1e9,
        },
        "roofline_fp64": {
            "bound": "fp64",
            "achieved": prof.get("fp64_instr_per_node", float("nan")) * nodes_local / (comb_ms * 1e-3),
            "peak": FP64_PEAK,
            "unit": "FP64 instr/s",
            "frac": prof.get("fp64_instr_per_node", float("nan")) * nodes_local / (comb_ms * 1e-3) / FP64_PEAK,
            "instr_per_node": prof.get("fp64_instr_per_node"),
            "source": "instr/node from ncu smsp__inst_executed_pipe_fp64.sum (profiles/ncu_summary.json); "
                      "peak from tools/fp64_peak.cu",
        },
        "e2e": {
            "value": e2e_value,
            "unit": UNIT,
            "h2d_bytes_per_step": 8 * nodes_local,
            "d2h_bytes_per_step": 8 * nodes_local,
            "steps": e2e_steps,
            "path": "lsg_solver_step_host per step: the full field H2D from pinned memory and the full result D2H, "
                    "chunked along z and overlapped with the stage kernels",
        },
        "e2e_leg": {
            "value": leg_value,
            "unit": UNIT,
            "steps": nst.value,
            "h2d_bytes_per_call": 8 * nodes_local,
            "d2h_bytes_per_call": 8 * nodes_local,
            "path": "one lsg_integrate call (the reference's integrate(term, {0, K*dt}, v0, {max_step}) usage, "
                    "as timed by the reference arm): pinned host field in, K steps, host field out",
        },
        "clocks": sampler.summary(),
    }
    if cpu_value is not None:
        line["cpu_baseline"] = {"value": cpu_value, "unit": UNIT, "cores": 1, "kind": "reference",
                                "sample": f"{cpu_info['steps']} RK3 steps of the full 101^3 Air3D workload, "
                                          f"1 thread, {cpu_info['seconds']:.1f} s (reference is single-threaded)"}
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dist-selftest", action="store_true",
                    help="under torchrun with one rank: run the multi-rank (NCCL) branch on a one-rank communicator")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    return b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
