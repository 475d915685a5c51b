"""Cell-centred finite differences of one subdomain (oracle).

Restates `/root/reference/pkg/src/helmsweep/discretization.py`:
  * ghost coefficients d = 1/h - tau/2, s = 1/h + tau/2, rhs = 1/(h^2 d)  -> :139-141
  * cell centres, origin (-side/2, -side/2)                                -> :75-77, :143-149
  * boundary cells per face, increasing global coordinate                  -> :151-158
  * staircase scatterer cells / owning subdomain                           -> :187-218
  * 5-point matrix with folded ghosts, identity Dirichlet rows              -> :221-256
  * SuperLU factorisation (scipy splu, default options)                    -> :171-174, :183-184
  * solve_local: traces scattered into the RHS, corners get two faces      -> :264-293
  * outgoing trace  -(u_g-u_c)/h - tau (u_g+u_c)/2                          -> :296-312
  * lifting solve with Dirichlet data -u_inc                               -> :315-332
  * mono-domain oracle                                                     -> :335-370

The matrix must come out bitwise identical to the reference's so that scipy's
SuperLU (the reference's third-party arithmetic, scipy>=1.10, unpinned:
pkg/pyproject.toml:12) produces identical factors; the diagonal is therefore
evaluated with the reference's operation order.
"""

from __future__ import annotations

from dataclasses import dataclass

import hashlib

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from .lattice import FACE_NAMES, FACE_STEP, Lattice

MONO_GUARD = 250_000


@dataclass(frozen=True)
class Problem:
    """Scattering problem (discretization.py:38-102).  `tau` defaults to i*kappa."""

    kappa: float
    n: int
    side: float
    center: tuple | None = None  # scatterer disk centre (reference frame), None = no scatterer
    radius: float = 0.0
    direction: tuple = (1.0, 0.0)
    tau: complex | None = None

    @property
    def h(self) -> float:
        return self.side / self.n

    @property
    def tau_c(self) -> complex:
        return complex(self.tau) if self.tau is not None else 1j * self.kappa

    @property
    def ghost(self):
        h, tau = self.h, self.tau_c
        d = 1.0 / h - tau / 2.0
        s = 1.0 / h + tau / 2.0
        return d, s

    def incident(self, x, y):
        dx, dy = self.direction
        nrm = np.hypot(dx, dy)
        return np.exp(1j * self.kappa * (dx * x + dy * y) / nrm)

    def cell_centres(self, a: int, b: int):
        o = -self.side / 2.0
        xs = o + (a - 1) * self.side + (np.arange(self.n) + 0.5) * self.h
        ys = o + (b - 1) * self.side + (np.arange(self.n) + 0.5) * self.h
        return np.meshgrid(xs, ys)

    def home(self, lat: Lattice):
        """Subdomain strictly containing the disk (discretization.py:203-218)."""
        if self.center is None:
            return None
        cx, cy = self.center
        r = self.radius
        o = -self.side / 2.0
        for a, b in lat.subs:
            x0, y0 = o + (a - 1) * self.side, o + (b - 1) * self.side
            if x0 < cx - r and cx + r < x0 + self.side and y0 < cy - r and cy + r < y0 + self.side:
                return (a, b)
        raise ValueError("scatterer must lie strictly inside one subdomain, away from interfaces")

    def dirichlet_cells(self, lat: Lattice, sub):
        if self.center is None or self.home(lat) != tuple(sub):
            return np.empty(0, dtype=np.intp)
        X, Y = self.cell_centres(*sub)
        cx, cy = self.center
        cells = np.flatnonzero(((X - cx) ** 2 + (Y - cy) ** 2 < self.radius ** 2).ravel())
        if cells.size == 0:
            raise ValueError("cells_per_side too coarse: no cell center inside the scatterer")
        return cells


def face_cells(n: int):
    """Boundary cell indices per face in W,S,N,E order (discretization.py:152-158)."""
    grid = np.arange(n * n).reshape(n, n)
    return (grid[:, 0].copy(), grid[0, :].copy(), grid[-1, :].copy(), grid[:, -1].copy())


def helmholtz_matrix(nx: int, ny: int, h: float, kappa: float, ratio: complex, dcells) -> sp.csr_matrix:
    """5-point operator with ghosts folded into the diagonal (discretization.py:221-256)."""
    ih2 = 1.0 / (h * h)
    N = nx * ny
    cell = np.arange(N).reshape(ny, nx)
    src = np.concatenate([cell[:, :-1].ravel(), cell[:, 1:].ravel(), cell[:-1, :].ravel(), cell[1:, :].ravel()])
    dst = np.concatenate([cell[:, 1:].ravel(), cell[:, :-1].ravel(), cell[1:, :].ravel(), cell[:-1, :].ravel()])
    nghost = np.zeros((ny, nx))
    nghost[0, :] += 1
    nghost[-1, :] += 1
    nghost[:, 0] += 1
    nghost[:, -1] += 1
    diag = 4.0 * ih2 - kappa * kappa - ih2 * ratio * nghost.ravel()
    isd = np.zeros(N, dtype=bool)
    isd[np.asarray(dcells, dtype=np.intp)] = True
    keep = ~isd[src]
    diag = np.where(isd, 1.0, diag)
    rows = np.concatenate([src[keep], np.arange(N)])
    cols = np.concatenate([dst[keep], np.arange(N)])
    vals = np.concatenate([np.full(int(keep.sum()), -ih2, dtype=complex), diag])
    return sp.csr_matrix((vals, (rows, cols)), shape=(N, N))


class Subdomain:
    """Factorised operator of one subdomain (discretization.py:116-184)."""

    def __init__(self, prob: Problem, lat: Lattice, sub, dcells=None, factor=True):
        self.sub = tuple(sub)
        self.prob = prob
        n, h = prob.n, prob.h
        self.n = n
        d, s = prob.ghost
        self.d, self.s = d, s
        self.rhs_coeff = 1.0 / (h * h * d)
        self.faces = face_cells(n)
        self.iface = [f for f, _ in lat.faces[self.sub]]  # interface faces, W,S,N,E order
        self.dcells = prob.dirichlet_cells(lat, sub) if dcells is None else np.asarray(dcells, dtype=np.intp)
        self.matrix = helmholtz_matrix(n, n, h, prob.kappa, s / d, self.dcells)
        self.lu = splu(self.matrix.tocsc()) if factor else None

    def factorise(self):
        self.lu = splu(self.matrix.tocsc())

    def matrix_key(self) -> str:
        """Digest of the exact CSC arrays handed to splu (shared-factor cache key)."""
        A = self.matrix.tocsc()
        h = hashlib.sha256()
        for arr in (A.data, A.indices, A.indptr, np.asarray(A.shape)):
            h.update(np.ascontiguousarray(arr).tobytes())
        return h.hexdigest()

    def solve(self, traces=None, source=None):
        """solve_local (discretization.py:264-293); traces: {face index: trace}."""
        n = self.n
        rhs = np.zeros(n * n, dtype=complex)
        for f, tr in (traces or {}).items():
            if f not in self.iface:
                raise ValueError(f"face {FACE_NAMES[f]} is not an interface face of {self.sub}")
            tr = np.asarray(tr, dtype=complex)
            if tr.shape != (n,):
                raise ValueError(f"trace has length {tr.size}, expected {n}")
            rhs[self.faces[f]] += self.rhs_coeff * tr
        if source is not None:
            if self.dcells.size == 0:
                raise ValueError(f"subdomain {self.sub} has no scatterer cells")
            rhs[self.dcells] = source
        return self.lu.solve(rhs)

    def outgoing(self, u, incoming, f):
        """extract_outgoing_trace (discretization.py:296-312)."""
        h, tau = self.prob.h, self.prob.tau_c
        uc = u[self.faces[f]]
        ug = (incoming + self.s * uc) / self.d
        return -(ug - uc) / h - tau * (ug + uc) / 2.0

    def lifting(self):
        """solve_lifting (discretization.py:315-332): (field, {face: trace})."""
        n = self.n
        if self.dcells.size == 0:
            return np.zeros(n * n, dtype=complex), {f: np.zeros(n, dtype=complex) for f in self.iface}
        X, Y = self.prob.cell_centres(*self.sub)
        data = -self.prob.incident(X.ravel()[self.dcells], Y.ravel()[self.dcells])
        w = self.solve(source=data)
        z = np.zeros(n, dtype=complex)
        return w, {f: self.outgoing(w, z, f) for f in self.iface}


def mono_solve(prob: Problem, lat: Lattice) -> np.ndarray:
    """Single-domain solution on the union grid (discretization.py:335-370)."""
    n = prob.n
    nx, ny = lat.n1 * n, lat.n2 * n
    if nx * ny > MONO_GUARD:
        raise ValueError(f"mono solve guard exceeded: {nx * ny} unknowns > {MONO_GUARD}")
    h = prob.h
    d, s = prob.ghost
    o = -prob.side / 2.0
    X, Y = np.meshgrid(o + (np.arange(nx) + 0.5) * h, o + (np.arange(ny) + 0.5) * h)
    rhs = np.zeros(nx * ny, dtype=complex)
    cells = np.empty(0, dtype=np.intp)
    if prob.center is not None:
        prob.home(lat)
        cx, cy = prob.center
        cells = np.flatnonzero(((X - cx) ** 2 + (Y - cy) ** 2 < prob.radius ** 2).ravel())
        if cells.size == 0:
            raise ValueError("cells_per_side too coarse: no cell center inside the scatterer")
        rhs[cells] = -prob.incident(X.ravel()[cells], Y.ravel()[cells])
    A = helmholtz_matrix(nx, ny, h, prob.kappa, s / d, cells)
    return splu(A.tocsc()).solve(rhs).reshape(ny, nx)
