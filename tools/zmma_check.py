"""Multi-RHS DMMA applies vs the single-RHS kernels, one line per (R, mode):
   python tools/zmma_check.py CFG R [R ...]   (env: HS_ZMMA2, HS_ZMMA2_KS)"""
import os
import sys

import numpy as np

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import cvec, product_problem, relerr
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig

c = CONFIGS[int(sys.argv[1])]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
L = s.layout.size
env = {k: v for k, v in os.environ.items() if k.startswith("HS_")}
for R in map(int, sys.argv[2:]):
    X = cvec(3, L, R)
    Y = s.apply_interface_operator(X)
    Z = s.bsp_apply(X)
    F = s.forward_sweep(X)
    ey, ez, ef = 0.0, 0.0, 0.0
    for r in range(R):
        x = np.ascontiguousarray(X[:, r])
        ey = max(ey, relerr(Y[:, r], s.apply_interface_operator(x)))
        ez = max(ez, relerr(Z[:, r], s.bsp_apply(x)))
        ef = max(ef, relerr(F[:, r], s.forward_sweep(x)))
    print(f"R={R} env={env} ims={ey:.2e} bsp={ez:.2e} fwd={ef:.2e}", flush=True)
