"""Order-of-accuracy study on the device kernels (runner.cpp:298-341,
acceptance criterion 1).  Inputs and truth come from the C library's sin/cos
(math.sin is glibc's, like the reference), derivatives from lsg_upwind."""
from __future__ import annotations

import math

import numpy as np

from . import abi


def convergence_study(ctx, scheme, refinements, profile="sin"):
    """Rows (n, dx, max_error, order) exactly as runner.cpp:298-341 builds them."""
    if refinements < 1:
        raise ValueError("convergence_study: refinements must be at least 1")
    if profile not in ("sin", "linear"):
        raise ValueError(f"convergence_study: unknown profile '{profile}' (valid: sin, linear)")
    periodic = profile == "sin"
    two_pi = 2.0 * math.pi
    rows = []
    for level in range(refinements + 1):
        n = 32 << level
        g = abi.make_grid([0.0], [1.0 - 1.0 / n if periodic else 1.0], [n], (0,) if periodic else ())
        dx = ((1.0 - 1.0 / n if periodic else 1.0) - 0.0) / (n - 1)
        axis = [0.0 + i * dx for i in range(n)]
        v = np.array([math.sin(two_pi * x) if periodic else x for x in axis])
        L, R = ctx.upwind(g, v, 0, scheme)
        err = 0.0
        for i, x in enumerate(axis):
            truth = two_pi * math.cos(two_pi * x) if periodic else 1.0
            err = max(err, abs(L[i] - truth))
            err = max(err, abs(R[i] - truth))
        order = math.nan if not rows else math.log2(rows[-1][2] / err)
        rows.append((n, dx, err, order))
    return rows
