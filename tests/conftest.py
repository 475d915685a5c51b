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


# HS_LIB=debug runs the whole GPU suite on the device-checks library: after
# every GPU test the first bounds / watchdog failure since the previous test
# (hs_debug_check) must be zero.  The check needs a context for its stream and
# device; the failure records are per process, so one small context serves.
_DBG = {}


@pytest.fixture(autouse=True)
def _device_checks(request):
    yield
    if os.environ.get("HS_LIB") != "debug" or request.node.get_closest_marker("gpu") is None:
        return
    import ctypes as C

    import torch
    if not torch.cuda.is_available():
        return
    if "sys" not in _DBG:
        from paper_2209_10886_b200.configs import small_case
        from paper_2209_10886_b200.interface_system import GpuInterfaceSystem
        spec, part = product_problem(small_case(2, 2, 8))
        _DBG["sys"] = GpuInterfaceSystem(spec, part)
    first, en = C.c_uint64(0), C.c_int(0)
    _DBG["sys"].ctx.call("hs_debug_check", C.byref(first), C.byref(en))
    assert en.value == 1, "HS_LIB=debug but the release library is loaded"
    assert first.value == 0, f"device check failed: unit {first.value >> 48}, line {(first.value >> 8) & 0xFFFFFFFF}, tag {first.value & 0xFF}"
