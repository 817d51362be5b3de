"""Problem descriptors of the BASELINE.json configs and the reference's own problems.

Each builder returns a ``Setup`` of plain descriptors (grid, problem, method,
tspan, initial-condition recipe); nothing here computes.  The synthetic
inputs follow SURVEY.md §8(d).

* rockets / rotation are the reference's own problems
  (reachability.cpp:68-133: build_rocket_problem, rigid_rotation_problem).
* cfg1..cfg5 are the BASELINE configs; their Hamiltonians are builder-defined
  and plugged through the reference's plugin API by the oracle
  (oracle/ref_driver.cpp) and as device kinds here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from . import abi

SPHERE, CYLINDER, PAIR_DISTANCE = 0, 1, 2


@dataclass
class Setup:
    name: str
    grid: abi.LsgGrid
    problem: abi.LsgProblem
    method: int
    tspan: tuple
    ic: tuple  # (shape, center, radius, ignored_dims)
    n_checkpoints: int = 2
    notes: dict = field(default_factory=dict)


def _grid(mins, maxs, counts, periodic=()):
    return abi.make_grid(mins, maxs, counts, periodic)


def cfg1_circle(n=101):
    """2-D circle SDF under constant convection, ENO2 + odeCFL2 (configs[0])."""
    g = _grid([-1.0, -1.0], [1.0, 1.0], [n, n])
    p = abi.make_problem(abi.HAM_LINEAR, abi.SCHEME_ENO2, abi.linear_params([1.0, 0.5]))
    return Setup("cfg1_circle_2d", g, p, abi.CFL2, (0.0, 0.5), (SPHERE, [-0.25, 0.0], 0.5, ()))


def cfg2_air3d(n=101, z_scale=1):
    """Air3D pursuit-evasion BRT, ENO3 LF + TVD-RK3, heading periodic (configs[1]).

    z_scale > 1 extends the heading axis to n*z_scale planes over the same
    period (weak scaling along the slab axis)."""
    nz = n * z_scale
    g = _grid([-6.0, -10.0, 0.0], [20.0, 10.0, 2.0 * math.pi * (nz - 1) / nz], [n, n, nz], periodic=(2,))
    p = abi.make_problem(abi.HAM_AIR3D, abi.SCHEME_ENO3, [5.0, 5.0, 1.0, 1.0], direction=abi.GROW,
                         restrict_update=True)
    return Setup("cfg2_air3d", g, p, abi.CFL3, (0.0, 2.8), (CYLINDER, [0.0, 0.0, 0.0], 5.0, (2,)))


def cfg3_dblint4(n=81):
    """4-D double-integrator pair BRT, WENO5 LF + RK3 (configs[2])."""
    g = _grid([-1.0] * 4, [1.0] * 4, [n] * 4)
    p = abi.make_problem(abi.HAM_DBLINT4, abi.SCHEME_WENO5, [], direction=abi.GROW, restrict_update=True)
    return Setup("cfg3_dblint4", g, p, abi.CFL3, (0.0, 0.5), (SPHERE, [0.0] * 4, 0.5, ()))


def cfg4_dubins6(n=41, scheme=abi.SCHEME_WENO5):
    """6-D two-vehicle Dubins game, both headings periodic (configs[3])."""
    two_pi = 2.0 * math.pi
    mins = [-1.0, -1.0, -math.pi, -1.0, -1.0, -math.pi]
    maxs = [1.0, 1.0, -math.pi + two_pi * (n - 1) / n, 1.0, 1.0, -math.pi + two_pi * (n - 1) / n]
    g = _grid(mins, maxs, [n] * 6, periodic=(2, 5))
    p = abi.make_problem(abi.HAM_DUBINS6, scheme, [], direction=abi.GROW, restrict_update=True)
    return Setup("cfg4_dubins6", g, p, abi.CFL3, (0.0, 0.5), (PAIR_DISTANCE, [0.0] * 6, 0.25, ()))


def cfg5_normal(n=512, scheme=abi.SCHEME_WENO5, z_scale=1, nz=None):
    """3-D motion in the normal direction on a periodic box (configs[4]; the
    reference has no curvature operator, so only the |grad v| term).

    z_scale > 1 stacks z_scale boxes along z (weak scaling: 512 x 512 x 512*N);
    nz overrides the plane count at the same spacing (a thin periodic slab of
    the same lines and strides, the CPU baseline's bounded sample)."""
    nz = n * z_scale if nz is None else nz
    h = 2.0 / n
    g = _grid([-1.0, -1.0, -1.0], [1.0 - h, 1.0 - h, -1.0 + h * (nz - 1)], [n, n, nz], periodic=(0, 1, 2))
    p = abi.make_problem(abi.HAM_NORMAL, scheme, [1.0])
    return Setup("cfg5_normal", g, p, abi.CFL3, (0.0, 0.25), (SPHERE, [0.0, 0.0, -1.0 + h * (nz // 2)], 0.5, ()))


def rockets(n=50, theta_periodic=False):
    """build_rocket_problem (reachability.cpp:68-103) + the acceptance solve
    (acceptance.cpp:381-419: N=50, tspan (-2.5, 0), 11 checkpoints, Cfl3)."""
    if theta_periodic:
        half_pi = math.pi / 2.0
        dtheta = math.pi / n
        g = _grid([-64.0, -64.0, -half_pi], [64.0, 64.0, half_pi - dtheta], [n, n, n], periodic=(2,))
    else:
        g = _grid([-64.0] * 3, [64.0] * 3, [n] * 3)
    # RocketParams defaults (reachability.hpp:18-24): a, g, capture_radius, u_min, u_max
    p = abi.make_problem(abi.HAM_ROCKETS, abi.SCHEME_ENO2, [1.0, 32.0, 1.5, -1.0, 1.0], direction=abi.GROW,
                         restrict_update=True)
    return Setup("rockets", g, p, abi.CFL3, (-2.5, 0.0), (CYLINDER, [0.0, 0.0, 0.0], 1.5, (2,)), n_checkpoints=11)


def rotation(n=101):
    """rigid_rotation_problem (reachability.cpp:105-133)."""
    g = _grid([-1.0, -1.0], [1.0, 1.0], [n, n])
    p = abi.make_problem(abi.HAM_ROTATION, abi.SCHEME_WENO5, [])
    return Setup("rotation", g, p, abi.CFL3, (0.0, 2.0 * math.pi), (SPHERE, [0.5, 0.0], 0.5, ()))


CONFIGS = {
    "cfg1": cfg1_circle,
    "cfg2": cfg2_air3d,
    "cfg3": cfg3_dblint4,
    "cfg4": cfg4_dubins6,
    "cfg5": cfg5_normal,
    "rockets": rockets,
    "rotation": rotation,
}
