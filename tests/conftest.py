import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs libhsb200 kernels)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path, allow_pickle=False)


def cvec(seed, size, R=None):
    rng = np.random.default_rng(seed)
    shape = (size,) if R is None else (size, R)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d > 0 else 1.0)


def oracle_problem(c):
    """oracle.Problem + Lattice for a config dict (paper_2209_10886_b200.configs)."""
    from oracle import Lattice, Problem
    ang = c["angle"] if c["angle"] is not None else 0.0
    prob = Problem(kappa=c["kappa"], n=c["n"], side=c["side"],
                   center=None if c["center"] is None else tuple(c["center"]), radius=c["radius"],
                   direction=(float(np.cos(ang)), float(np.sin(ang))))
    return prob, Lattice(c["n1"], c["n2"])


def product_problem(c):
    from paper_2209_10886_b200.discretization import ProblemSpec, Scatterer
    from paper_2209_10886_b200.indexing import Partition
    ang = c["angle"] if c["angle"] is not None else 0.0
    spec = ProblemSpec(kappa=c["kappa"], cells_per_side=c["n"], subdomain_side=c["side"],
                       scatterer=None if c["center"] is None else Scatterer(tuple(c["center"]), c["radius"]),
                       incident_direction=(float(np.cos(ang)), float(np.sin(ang))))
    return spec, Partition(c["n1"], c["n2"])
