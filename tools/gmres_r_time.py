"""GMRES with R right-hand sides (config 4 by default): time-to-solution
(median of three), iterations, and the solution's difference between the
one-reduction Arnoldi (default) and the cooperative MGS kernel
(HS_ARNOLDI_R=mgs in a second process; this script runs one mode).
    python tools/gmres_r_time.py [CFG] [out.npy]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS, angles  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[k]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
b = s.rhs(directions=[(float(np.cos(t)), float(np.sin(t))) for t in angles(c)])
s.gmres(b, "bsp", tol=c["tol"], maxit=1000)
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = s.gmres(b, "bsp", tol=c["tol"], maxit=1000)
    ts.append(time.perf_counter() - t0)
x = np.asarray(res.solution)
resid = np.linalg.norm(s.apply_interface_operator(x) - b, axis=0) / np.linalg.norm(b, axis=0)
print({"config": k, "gmres_s": sorted(ts)[1], "iterations": [int(min(res.iterations)), int(max(res.iterations))],
       "max_true_residual": float(resid.max())})
if len(sys.argv) > 2:
    np.save(sys.argv[2], x)
