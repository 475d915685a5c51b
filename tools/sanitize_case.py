"""One small workload per dataflow kernel, for compute-sanitizer runs
(tools/sanitize.sh): python tools/sanitize_case.py CASE

  tma     k_bsp_tma (map-once fused BSP apply + GMRES A M v), small 3x3 + cfg1
  fused   k_bsp_fused (register-streaming fused kernel, HS_FUSED_TMA=0)
  zmma    k_zmma (4 RHS per-step DMMA contraction) + shared-map variant
  gmres   GMRES on cfg1 (k_mgs1c cluster Arnoldi) and the grid Arnoldi (forced)
Each result is checked against the plain per-step path, so a run that
completes under a tool also proves the instrumented kernels computed the same.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import cvec, product_problem, relerr  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS, small_case  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

case = sys.argv[1]
cases = [small_case(3, 3, 32), CONFIGS[1]]
for c in cases:
    spec, part = product_problem(c)
    ref = GpuInterfaceSystem(spec, part, fused="literal", sweep=SweepConfig(blocks=c["blocks"]))
    L = ref.layout.size
    if case in ("tma", "fused"):
        s = GpuInterfaceSystem(spec, part, fused=True, sweep=SweepConfig(blocks=c["blocks"]))
        g = cvec(3, L)
        for _ in range(3):
            assert relerr(s.bsp_apply(g), ref.bsp_apply(g)) < 1e-13
        b = s.rhs()
        r1, r2 = s.gmres(b, "bsp", tol=1e-8, maxit=100), ref.gmres(b, "bsp", tol=1e-8, maxit=100)
        assert r1.iterations == r2.iterations and relerr(r1.solution, r2.solution) < 1e-11
    elif case == "zmma":
        for maps in ("subdomain", "shared"):
            s = GpuInterfaceSystem(spec, part, fused=False, maps=maps, sweep=SweepConfig(blocks=c["blocks"]))
            G = cvec(5, L, 4)
            Z = s.bsp_apply(G)
            for r in range(4):
                assert relerr(Z[:, r], ref.bsp_apply(np.ascontiguousarray(G[:, r]))) < 1e-12
            assert relerr(s.apply_interface_operator(G)[:, 1],
                          ref.apply_interface_operator(np.ascontiguousarray(G[:, 1]))) < 1e-12
    elif case == "gmres":
        b = ref.rhs()
        for mode in ("auto", "grid", "cgs2"):
            s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
            r1 = s.gmres(b, "bsp", tol=1e-8, maxit=100, arnoldi=mode)
            r2 = ref.gmres(b, "bsp", tol=1e-8, maxit=100)
            assert abs(r1.iterations - r2.iterations) <= 1 and relerr(r1.solution, r2.solution) < 1e-8
    else:
        raise SystemExit(f"unknown case {case}")
print(f"sanitize case {case}: OK")
