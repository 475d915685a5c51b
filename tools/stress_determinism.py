"""Stress: repeated fused applies (BSP and GMRES's A M v) must be bitwise
reproducible -- a missed dependency in the dataflow kernels would show up as
an occasional different z.  python tools/stress_determinism.py CFG N [R]
(R > 1: the R-RHS DMMA dataflow apply k_zmma2_df and the batched GMRES)"""
import hashlib
import sys

import torch

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import cvec, product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig

cfg, N = int(sys.argv[1]), int(sys.argv[2])
R = int(sys.argv[3]) if len(sys.argv) > 3 else 1
c = CONFIGS[cfg]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
g = torch.from_numpy(cvec(7, s.layout.size, R if R > 1 else None)).cuda()
ref = hashlib.sha1(s.bsp_apply(g).cpu().numpy().tobytes()).hexdigest()
bad = 0
for i in range(N):
    if hashlib.sha1(s.bsp_apply(g).cpu().numpy().tobytes()).hexdigest() != ref:
        bad += 1
if R > 1:
    import math
    from paper_2209_10886_b200.configs import angles
    b = s.rhs(directions=[(math.cos(t), math.sin(t)) for t in angles(c)][:R]) if c["nrhs"] > 1 else s.rhs()
else:
    b = s.rhs()
r0 = s.gmres(b, "bsp", tol=1e-6, maxit=1000)
x0 = hashlib.sha1(r0.solution.tobytes()).hexdigest()
gb = 0
for i in range(max(1, N // 50)):
    r = s.gmres(b, "bsp", tol=1e-6, maxit=1000)
    if hashlib.sha1(r.solution.tobytes()).hexdigest() != x0 or r.iterations != r0.iterations:
        gb += 1
print(f"cfg{cfg} R={R}: {N} BSP applies, {bad} differing; {max(1, N // 50)} GMRES solves, {gb} differing", flush=True)
