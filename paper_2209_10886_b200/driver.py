"""End-to-end solve with the SPEC driver API (not shipped by
the reference): lifting -> b -> GMRES((I - S), M) -> u_i = v_i + w_i ->
stitched field, all on the GPU.  `wall_time` is the GMRES phase only
(SPEC.md:440).  The mono-domain solve is a CPU oracle (discretization.py:
335-370, size-guarded) and is not part of the product: pass its field as
`mono` to get `error_vs_mono`.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .interface_system import GmresOptions, GpuInterfaceSystem, SweepConfig


@dataclass
class SolveReport:
    """SPEC.md:431-434."""

    iterations: int
    steps_per_iteration: int
    total_sequential_steps: int
    residual_history: list
    wall_time: float
    converged: bool
    schedule: list = field(default_factory=list)
    error_vs_mono: dict | None = None
    field: np.ndarray | None = None
    solution: np.ndarray | None = None
    setup_time: float = 0.0


def compare_with_mono(stitched: np.ndarray, mono: np.ndarray) -> dict:
    """relative max-norm and L2 differences."""
    u, v = np.asarray(stitched), np.asarray(mono)
    if u.shape != v.shape:
        raise ValueError(f"grid mismatch: {u.shape} vs {v.shape}")
    vmax = np.abs(v).max()
    vl2 = np.linalg.norm(v)
    return {"max_rel": float(np.abs(u - v).max() / vmax) if vmax > 0 else float(np.abs(u - v).max()),
            "l2_rel": float(np.linalg.norm(u - v) / vl2) if vl2 > 0 else float(np.linalg.norm(u - v))}


def solve_problem(spec, partition, sweep_config: SweepConfig | None = None,
                  gmres_options: GmresOptions | None = None, run_mono_check: bool = False,
                  mono: np.ndarray | None = None, device: int = 0, maps: str = "subdomain",
                  reconstruct: bool = True) -> SolveReport:
    """SPEC.md:437-444 on the GPU."""
    sweep_config = sweep_config or SweepConfig()
    gmres_options = gmres_options or GmresOptions()
    if run_mono_check and mono is None:
        raise ValueError("run_mono_check needs the mono-domain field (the mono solve is a CPU oracle)")
    t0 = time.perf_counter()
    system = GpuInterfaceSystem(spec, partition, device=device, sweep=sweep_config, maps=maps)
    setup = time.perf_counter() - t0
    b = system.assemble_rhs(system.compute_liftings())
    res = system.gmres(b, sweep_config.kind, tol=gmres_options.tol, maxit=gmres_options.maxit)
    sched = system.step_schedule(sweep_config.kind) if sweep_config.kind != "none" else []
    spi = len(sched)
    rep = SolveReport(iterations=res.iterations, steps_per_iteration=spi,
                      total_sequential_steps=res.iterations * spi, residual_history=res.history,
                      wall_time=res.wall_time, converged=res.converged, schedule=sched,
                      solution=res.solution, setup_time=setup)
    if reconstruct or run_mono_check:
        rep.field = system.reconstruct_solution(res.solution)
        if mono is not None:
            rep.error_vs_mono = compare_with_mono(rep.field, mono)
    return rep
