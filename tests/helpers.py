"""Shared test helpers: oracle-side initial conditions and random fields."""
import numpy as np

from paper_2507_11542_b200 import abi
from paper_2507_11542_b200 import problems as P


def node_count(g):
    n = 1
    for d in range(g.dim):
        n *= g.counts[d]
    return n


def coords(checker, g):
    """Column-major coordinate fields (grid.cpp:54-64) from the checker's axes."""
    axes = [checker.axis(g, d) for d in range(g.dim)]
    mesh = np.meshgrid(*axes, indexing="ij")
    return [m.transpose(tuple(range(g.dim - 1, -1, -1))).ravel() for m in mesh]


def initial_value(checker, setup):
    """Initial field through the reference's own implicit surfaces
    (implicit_surfaces.cpp:20-71); the cfg4 pair distance is builder-defined."""
    shape, center, radius, ignored = setup.ic
    g = setup.grid
    if shape == P.SPHERE:
        return checker.sphere(g, center, radius)
    if shape == P.CYLINDER:
        return checker.cylinder(g, ignored, center, radius)
    x = coords(checker, g)
    a = x[0] - x[3]
    b = x[1] - x[4]
    r2 = 0.0 + a * a
    r2 = r2 + b * b
    return np.sqrt(r2) - radius


def random_field(g, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, node_count(g))


def small(name):
    """Oracle-sized versions of each config."""
    return {
        "cfg1": dict(n=41),
        "cfg2": dict(n=21),
        "cfg3": dict(n=11),
        "cfg4": dict(n=7),
        "cfg5": dict(n=24),
        "rockets": dict(n=20),
        "rotation": dict(n=41),
    }[name]
