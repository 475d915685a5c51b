"""End-to-end driver (oracle restatement of SPEC.md:426-480; not shipped by
the reference): lifting -> b -> GMRES((I-S), M) -> u_i = v_i + w_i -> stitch ->
compare with the mono-domain solve (discretization.py:335-370)."""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .fd import Problem, mono_solve
from .gmres import gmres
from .interface import Interface
from .lattice import Lattice
from .sweeps import Preconditioner


@dataclass
class Report:
    iterations: int
    converged: bool
    history: list
    wall_time: float
    x: np.ndarray
    b: np.ndarray
    field: np.ndarray | None = None
    error_vs_mono: dict | None = None
    steps_per_iteration: int = 0


def reconstruct(itf: Interface, g, lifts):
    """Per-subdomain v_i + w_i stitched on the union grid."""
    lat, n = itf.lat, itf.n
    out = np.zeros((lat.n2 * n, lat.n1 * n), dtype=complex)
    for s in lat.subs:
        op = itf.ops[s]
        tr = {f: g[itf.block(lat.m_index(s, j))] for f, j in lat.faces[s]}
        v = op.solve(tr) if tr else np.zeros(n * n, complex)
        w, _ = lifts[s]
        a, b = s
        out[(b - 1) * n:b * n, (a - 1) * n:a * n] = (v + w).reshape(n, n)
    return out


def compare(u, v):
    """compare_with_mono."""
    if u.shape != v.shape:
        raise ValueError("grid mismatch")
    return {"max_rel": float(np.abs(u - v).max() / np.abs(v).max()),
            "l2_rel": float(np.linalg.norm(u - v) / np.linalg.norm(v))}


def solve_problem(prob: Problem, lat: Lattice, kind="bsp", tol=1e-6, maxit=1000,
                  mono_check=False, blocks=None, seam="dedup", backend="superlu",
                  reconstruct_field=False):
    itf = Interface(prob, lat, backend=backend)
    lifts = itf.liftings() if backend == "superlu" else None
    if backend == "superlu":
        b = itf.rhs(lifts)
    else:
        from .schur import lifting_traces
        home, tr = lifting_traces(prob, lat)
        b = np.zeros(itf.size, dtype=complex)
        if home is not None:
            for f, j in lat.faces[home]:
                b[itf.block(lat.m_index(j, home))] = tr[f]
    pc = Preconditioner(itf, kind, seam=seam, blocks=blocks)
    t0 = time.perf_counter()
    res = gmres(itf.apply_A, None if kind == "none" else pc, b, tol=tol, maxit=maxit)
    wall = time.perf_counter() - t0
    rep = Report(res.iterations, res.converged, res.history, wall, res.x, b,
                 steps_per_iteration=pc.steps_per_apply if kind != "none" else 0)
    if (reconstruct_field or mono_check) and backend == "superlu":
        rep.field = reconstruct(itf, res.x, lifts)
        if mono_check:
            rep.error_vs_mono = compare(rep.field, mono_solve(prob, lat))
    return rep
