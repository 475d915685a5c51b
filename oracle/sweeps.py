"""Sweeping preconditioners SP and BSP (oracle restatement of SPEC.md).

The reference ships no preconditioner module; this follows the specification:
  * forward_sweep / backward_sweep, z|gamma += S_{gamma,gamma-1} z|gamma-1    -> SPEC.md:306-321
  * sgs_apply = backward(forward(r)), 2(N_g-1) steps                          -> SPEC.md:322-330
  * bj_half_apply: concurrent in-window substitutions, dedup / literal seams  -> SPEC.md:331-339, 367-371
  * bsp_apply with the intermediate residual r' = b - (I-S) z_L              -> SPEC.md:340-348
  * step_schedule / StepTrace text format                                    -> SPEC.md:300-303, 349-357, 375
Every S application goes through `Interface.restricted` / `Interface.apply_A`
(the restatement of interface_system.py:144-162).
"""

from __future__ import annotations

import numpy as np

from .interface import Interface
from .lattice import windows as make_windows


def _run(gen):
    """Drive a stage generator to completion and return its value."""
    while True:
        try:
            next(gen)
        except StopIteration as stop:
            return stop.value


def _mask(itf: Interface, groups):
    """Boolean mask over vector entries owned by the given groups
    (TraceLayout.group_indices, interface_system.py:48-56)."""
    g = np.repeat(np.asarray(itf.lat.block_group()), itf.n)
    return np.isin(g, list(groups))


class Preconditioner:
    def __init__(self, itf: Interface, kind: str = "bsp", seam: str = "dedup",
                 intermediate_residual: bool = True, count_residual_steps: bool = False,
                 blocks: int | None = None):
        if kind not in ("none", "sp", "bsp"):
            raise ValueError(kind)
        if seam not in ("dedup", "literal"):
            raise ValueError(seam)
        self.itf, self.kind, self.seam = itf, kind, seam
        self.inter = intermediate_residual
        self.count_res = count_residual_steps
        lat = itf.lat
        self.ng = lat.n_groups
        self.lower = make_windows(lat.n1, lat.n2, "lower", blocks)
        self.upper = make_windows(lat.n1, lat.n2, "upper", blocks)

    # ---- SP
    def forward_sweep(self, r):
        z = np.array(r, dtype=complex, copy=True)
        for gam in range(3, self.ng + 2):
            z += self.itf.restricted(z, {gam - 1}, {gam})
        return z

    def backward_sweep(self, r):
        z = np.array(r, dtype=complex, copy=True)
        for gam in range(self.ng, 1, -1):
            z += self.itf.restricted(z, {gam + 1}, {gam})
        return z

    def sgs_apply(self, r):
        return self.backward_sweep(self.forward_sweep(r))

    # ---- BSP
    # The *_iter forms yield after every S application (one restricted_apply or
    # apply_interface_operator call of the reference) so that a caller can run
    # an apply stage by stage (bench.py's bounded CPU-baseline samples); the
    # plain forms run them to completion -- one implementation of the arithmetic.
    def _window_solve_iter(self, r, lo, hi, direction):
        zw = np.where(_mask(self.itf, range(lo, hi + 1)).reshape((-1,) + (1,) * (np.ndim(r) - 1)), r, 0)
        zw = zw.astype(complex)
        if direction == "forward":
            for gam in range(lo + 1, hi + 1):
                zw += self.itf.restricted(zw, {gam - 1}, {gam})
                yield
        else:
            for gam in range(hi - 1, lo - 1, -1):
                zw += self.itf.restricted(zw, {gam + 1}, {gam})
                yield
        return zw

    def bj_half_apply_iter(self, r, direction):
        r = np.asarray(r, dtype=complex)
        wins = self.lower if direction == "forward" else self.upper
        if self.seam == "dedup":
            z = r.copy()
            for lo, hi in wins:
                m = _mask(self.itf, range(lo, hi + 1)).reshape((-1,) + (1,) * (r.ndim - 1))
                zw = yield from self._window_solve_iter(r, lo, hi, direction)
                z += zw - np.where(m, r, 0)
            return z
        z = np.zeros_like(r)
        for lo, hi in wins:
            z += yield from self._window_solve_iter(r, lo, hi, direction)
        return z

    def bsp_apply_iter(self, b):
        b = np.asarray(b, dtype=complex)
        zL = yield from self.bj_half_apply_iter(b, "forward")
        if self.inter:
            rp = b - self.itf.apply_A(zL)
            yield
        else:
            rp = b
        zU = yield from self.bj_half_apply_iter(rp, "backward")
        return zL + zU

    def _window_solve(self, r, lo, hi, direction):
        return _run(self._window_solve_iter(r, lo, hi, direction))

    def bj_half_apply(self, r, direction):
        return _run(self.bj_half_apply_iter(r, direction))

    def bsp_apply(self, b):
        return _run(self.bsp_apply_iter(b))

    def __call__(self, r):
        if self.kind == "none":
            return np.array(r, dtype=complex, copy=True)
        if self.kind == "sp":
            return self.sgs_apply(r)
        return self.bsp_apply(r)

    @property
    def steps_per_apply(self) -> int:
        return len(step_schedule(self))


def step_schedule(pc: Preconditioner):
    """[(step, phase, [subdomains])] the sweeps execute."""
    lat = pc.itf.lat if hasattr(pc, "itf") else pc.lat
    groups = lat.groups
    recs = []
    if pc.kind == "none" or lat.n_groups < 2:
        return recs
    if pc.kind == "sp":
        fw = [[gam - 1] for gam in range(3, pc.ng + 2)]
        bw = [[gam + 1] for gam in range(pc.ng, 1, -1)]
        res = []
    else:
        depth_f = max(hi - lo for lo, hi in pc.lower)
        fw = [[lo + t - 1 for lo, hi in pc.lower if t <= hi - lo] for t in range(1, depth_f + 1)]
        depth_b = max(hi - lo for lo, hi in pc.upper)
        bw = [[hi - t + 1 for lo, hi in pc.upper if t <= hi - lo] for t in range(1, depth_b + 1)]
        res = [list(groups)] if (pc.inter and pc.count_res) else []
    step = 0
    for phase, seq in (("forward", fw), ("residual", res), ("backward", bw)):
        for gs in seq:
            step += 1
            subs = [s for gam in sorted(set(gs)) for s in groups.get(gam, [])]
            recs.append((step, phase, subs))
    return recs


class SchedulePlan:
    """Schedule-only view of a preconditioner (no operators): for step counts
    and wavefront records without factorising anything."""

    def __init__(self, lat, kind="bsp", blocks=None, intermediate_residual=True, count_residual_steps=False):
        self.lat, self.kind = lat, kind
        self.ng = lat.n_groups
        self.inter, self.count_res = intermediate_residual, count_residual_steps
        self.lower = make_windows(lat.n1, lat.n2, "lower", blocks)
        self.upper = make_windows(lat.n1, lat.n2, "upper", blocks)


def format_trace(recs) -> str:
    """StepTrace text lines."""
    return "".join(
        f"step={t} phase={ph} solves=" + ";".join(f"({a},{b})" for a, b in subs) + "\n"
        for t, ph, subs in recs)
