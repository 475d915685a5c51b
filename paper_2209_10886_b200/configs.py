"""The BASELINE.json configurations in the reference's coordinates.

The reference fixes the origin at (-side/2, -side/2) (discretization.py:75-77),
so BASELINE's unit square [0,1]^2 is the reference domain translated by
(side/2, side/2); scatterer centres below are given in the reference frame
(SURVEY.md §8d).  tau = i*kappa everywhere (discretization.py:100-102).
"""

from __future__ import annotations

import math

import numpy as np


def _cfg(name, n1, n2, n, side, ppw, center, radius, angle, blocks, nrhs=1, tol=1e-6):
    h = side / n
    return dict(name=name, n1=n1, n2=n2, n=n, side=side, kappa=2.0 * math.pi / (ppw * h),
                center=center, radius=radius, angle=angle, blocks=blocks, nrhs=nrhs, tol=tol)


CONFIGS = {
    # 128x128 grid, 4x4 of n=32, 10 ppw, disk r=0.05 in subdomain (2,2), t=pi/4, 2 blocks
    1: _cfg("cfg1", 4, 4, 32, 0.25, 10, (0.25, 0.25), 0.05, math.pi / 4, None),
    # 512x512 grid, 8x8 of n=64, disk in (4,4); block count varied 1,2,4,8 (2 = reference rule)
    2: _cfg("cfg2", 8, 8, 64, 0.125, 10, (0.375, 0.375), 0.05, math.pi / 4, None),
    # 2048x2048 grid, 16x16 of n=128, r=0.02 in (8,8), t ~ U[0,2pi) from seed 0, 4 blocks
    3: _cfg("cfg3", 16, 16, 128, 0.0625, 10, (0.4375, 0.4375), 0.02,
            float(np.random.default_rng(0).uniform(0, 2 * math.pi)), 4),
    # config 2 with 64 right-hand sides t_k = 2 pi k / 64 (reference windows)
    4: _cfg("cfg4", 8, 8, 64, 0.125, 10, (0.375, 0.375), 0.05, None, None, nrhs=64),
    # [0,2]x[0,1], 8192x4096 grid, 32x16 of n=256, 8 ppw, r=0.03 in (16,8), t=0.3, 8 blocks
    5: _cfg("cfg5", 32, 16, 256, 0.0625, 8, (0.9375, 0.4375), 0.03, 0.3, 8),
}


def angles(cfg):
    """Incident angles of a config (64 for config 4)."""
    if cfg["nrhs"] > 1:
        return [2.0 * math.pi * k / cfg["nrhs"] for k in range(cfg["nrhs"])]
    return [cfg["angle"]]


def small_case(n1, n2, n, kappa=2 * math.pi, side=2.5, center=(0.0, 0.0), radius=1.0, angle=0.0,
               blocks=None):
    """Desk-scale case of SPEC.md (kappa = 2 pi, side 2.5, unit disk in (1,1))."""
    return dict(name=f"small_{n1}x{n2}_n{n}", n1=n1, n2=n2, n=n, side=side, kappa=kappa,
                center=center, radius=radius, angle=angle, blocks=blocks, nrhs=1, tol=1e-6)


def with_blocks(cfg, p):
    c = dict(cfg)
    c["blocks"] = p
    c["name"] = f"{cfg['name']}_p{p}"
    return c
