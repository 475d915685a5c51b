"""Dense interface-to-interface Schur maps (diagnostic accurate oracle).

For subdomain i the composition of solve_local (discretization.py:264-293)
and extract_outgoing_trace (discretization.py:296-312) is the linear map

    T_i = -(s/d) I - (2 tau / (h^3 d^2)) E^T A_i^{-1} E

from its incoming traces (faces W,S,N,E, m-order) to its outgoing traces,
where E selects the boundary cells of each face (corners belong to two faces)
and d, s are the ghost coefficients (discretization.py:139-140).

A_i is taken in Dirichlet-eliminated form: the identity rows of the scatterer
cells (discretization.py:247-251) are solved for first (u_D = f_D) and moved
to the right-hand side, so the factorised matrix is the symmetric principal
block A_FF.  This removes the badly scaled identity rows that make the
reference's SuperLU factor lose 1e-11..1e-9 on the scatterer subdomain
(SURVEY.md §7 hard part 1, §8c).  The arithmetic here is SciPy SuperLU on
A_FF -- independent of the GPU's block-tridiagonal elimination.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from .fd import Problem, face_cells, helmholtz_matrix
from .lattice import Lattice


def _split(prob: Problem, dcells):
    n = prob.n
    d, s = prob.ghost
    A = helmholtz_matrix(n, n, prob.h, prob.kappa, s / d, np.empty(0, dtype=np.intp)).tocsr()
    isd = np.zeros(n * n, dtype=bool)
    isd[np.asarray(dcells, dtype=np.intp)] = True
    free = np.flatnonzero(~isd)
    dir_ = np.flatnonzero(isd)
    AFF = A[free][:, free].tocsc()
    AFD = A[free][:, dir_].tocsr()
    return free, dir_, AFF, AFD


def boundary_response(prob: Problem, dcells, rhs_cols):
    """Solve the reference system (identity rows at Dirichlet cells) for dense
    RHS columns `rhs_cols` (n^2 x R) in eliminated form; returns u (n^2 x R)."""
    free, dir_, AFF, AFD = _split(prob, dcells)
    f = np.asarray(rhs_cols, dtype=complex)
    u = np.zeros_like(f)
    uD = f[dir_]
    u[dir_] = uD
    rhsF = f[free] - (AFD @ uD if dir_.size else 0)
    u[free] = splu(AFF).solve(np.ascontiguousarray(rhsF))
    return u


def schur_map(prob: Problem, dcells) -> np.ndarray:
    """Full 4n x 4n map (faces W,S,N,E) of a subdomain with Dirichlet cells `dcells`."""
    n, h = prob.n, prob.h
    d, s = prob.ghost
    tau = prob.tau_c
    faces = face_cells(n)
    E = np.zeros((n * n, 4 * n), dtype=complex)
    for q, cells in enumerate(faces):
        E[cells, q * n + np.arange(n)] = 1.0
    rhs_coeff = 1.0 / (h * h * d)
    u = boundary_response(prob, dcells, rhs_coeff * E)
    uc = np.concatenate([u[cells] for cells in faces], axis=0)  # 4n x 4n
    return -(s / d) * np.eye(4 * n) - (2.0 * tau / (h * d)) * uc


def compact(T4: np.ndarray, n: int, iface) -> np.ndarray:
    """Sub-block of the 4-face map on the interface faces `iface` (W,S,N,E indices)."""
    idx = np.concatenate([np.arange(f * n, (f + 1) * n) for f in iface])
    return T4[np.ix_(idx, idx)]


def schur_maps_for(prob: Problem, lat: Lattice, subs=None):
    """Compact T_i for the requested subdomains; only two distinct operators
    exist (generic and scatterer, discretization.py:224-229)."""
    subs = lat.subs if subs is None else subs
    home = prob.home(lat)
    cache = {}
    out = {}
    for s in subs:
        key = "scat" if s == home else "gen"
        if key not in cache:
            dc = prob.dirichlet_cells(lat, s) if key == "scat" else np.empty(0, dtype=np.intp)
            cache[key] = schur_map(prob, dc)
        out[s] = compact(cache[key], prob.n, [f for f, _ in lat.faces[s]])
    return out


def lifting_traces(prob: Problem, lat: Lattice, directions=None):
    """Outgoing lifting traces of the scatterer subdomain, eliminated form
    (discretization.py:315-332).  Returns (home, {face: trace (n,) or (n, R)})."""
    home = prob.home(lat)
    if home is None:
        return None, {}
    n, h = prob.n, prob.h
    d, _ = prob.ghost
    tau = prob.tau_c
    dc = prob.dirichlet_cells(lat, home)
    X, Y = prob.cell_centres(*home)
    xs, ys = X.ravel()[dc], Y.ravel()[dc]
    dirs = [prob.direction] if directions is None else directions
    f = np.zeros((n * n, len(dirs)), dtype=complex)
    for r, (dx, dy) in enumerate(dirs):
        nrm = np.hypot(dx, dy)
        f[dc, r] = -np.exp(1j * prob.kappa * (dx * xs + dy * ys) / nrm)
    u = boundary_response(prob, dc, f)
    faces = face_cells(n)
    tr = {}
    for q, _ in lat.faces[home]:
        v = -(2.0 * tau / (h * d)) * u[faces[q]]
        tr[q] = v[:, 0] if directions is None else v
    return home, tr
