"""Matrix-free interface operator S, (I - S) and restricted blocks (oracle).

Restates `/root/reference/pkg/src/helmsweep/interface_system.py`:
  * vector layout: 2 N_e blocks of n in m-order                 -> :30-62
  * one local solve per subdomain, outgoing traces per face     -> :115-133
  * S g, (I - S) g, V_T S V_Src^T g                             -> :135-162
  * liftings and right-hand side b                              -> :98-113
  * dense S oracle (size-guarded)                               -> :164-175

Two local-solve back ends:
  * "superlu": the reference arithmetic (SuperLU per subdomain), used for
    parity and as the timed CPU baseline;
  * "schur": dense Schur maps T_i built from the Dirichlet-eliminated operator
    (`oracle.schur`), the "diagnostic accurate oracle" of SURVEY.md §8c; it is
    what the GPU computes, and is fast enough for configs 3 and 5 on the CPU.
Vectors may be (L,) or (L, R) (R right-hand sides, RHS fastest).
"""

from __future__ import annotations

import numpy as np

from .fd import Problem, Subdomain
from .lattice import Lattice

DENSE_GUARD = 6000


class Interface:
    def __init__(self, prob: Problem, lat: Lattice, backend: str = "superlu", subs=None,
                 share_factors: bool = False):
        """`subs` optionally restricts which subdomains are factorised (spot checks
        at configs too large to factor every subdomain).  `share_factors` gives
        every subdomain whose matrix is bitwise identical to an earlier one that
        one's SuperLU object: `_assemble_grid` uses one ghost ratio on all four
        faces (discretization.py:224-229), so only the generic and the scatterer
        operator exist, and each solve is bit-for-bit the unshared one (SuperLU
        is deterministic; solves are read-only on the factor,
        discretization.py:119-123).  cfg5 then holds 2 factors instead of 512."""
        self.prob, self.lat, self.n = prob, lat, prob.n
        self.size = lat.n_pairs * prob.n
        self.backend = backend
        todo = lat.subs if subs is None else [tuple(s) for s in subs]
        self.home = prob.home(lat)
        if backend == "superlu":
            if share_factors:
                cache = {}
                self.ops = {}
                for s in todo:
                    op = Subdomain(prob, lat, s, factor=False)
                    key = op.matrix_key()
                    if key not in cache:
                        op.factorise()
                        cache[key] = op.lu
                    op.lu = cache[key]
                    op.matrix = None  # the shared factor is all a solve needs (512 x 7 MB at cfg5)
                    self.ops[s] = op
                self.n_factors = len(cache)
            else:
                self.ops = {s: Subdomain(prob, lat, s) for s in todo}
                self.n_factors = len(self.ops)
        elif backend == "schur":
            from .schur import schur_maps_for
            self.T = schur_maps_for(prob, lat, todo)
            self.ops = {s: Subdomain(prob, lat, s, factor=False) for s in todo}
        else:
            raise ValueError(backend)

    # ---- layout helpers (interface_system.py:36-56)
    def block(self, m: int) -> slice:
        return slice((m - 1) * self.n, m * self.n)

    def in_slice(self, s) -> slice:
        """Contiguous incoming blocks m(s, .) of subdomain s (its owned blocks)."""
        first = self.lat.first_block[s]
        k = len(self.lat.faces[s])
        return slice((first - 1) * self.n, (first - 1 + k) * self.n)

    def check(self, g):
        g = np.asarray(g)
        if g.shape[0] != self.size:
            raise ValueError(f"interface vector has length {g.shape[0]}, expected {self.size}")
        return g.astype(complex, copy=False)

    # ---- one subdomain (interface_system.py:115-133)
    def scatter_one(self, s, g, target_groups=None):
        """Outgoing blocks of subdomain s toward neighbours whose group is in
        target_groups (all when None): list of (slice, trace)."""
        lat, n = self.lat, self.n
        faces = lat.faces[s]
        outs = [(f, j) for f, j in faces if target_groups is None or (j[0] + j[1]) in target_groups]
        if not outs:
            return []
        x = g[self.in_slice(s)]
        if not np.any(x):
            return []
        res = []
        if self.backend == "superlu":
            op = self.ops[s]
            cols = x.reshape(len(faces), n, -1)
            R = cols.shape[2]
            for r in range(R):
                tr = {f: cols[q, :, r] for q, (f, _) in enumerate(faces)}
                u = op.solve(tr)
                for q, (f, j) in enumerate(faces):
                    if (f, j) in outs:
                        res.append((self.block(lat.m_index(j, s)), r, op.outgoing(u, tr[f], f)))
        else:
            T = self.T[s]
            y = T @ x.reshape(len(faces) * n, -1)
            for q, (f, j) in enumerate(faces):
                if (f, j) in outs:
                    res.append((self.block(lat.m_index(j, s)), None, y[q * n:(q + 1) * n]))
        return res

    def _write(self, out, writes):
        for sl, r, tr in writes:
            if r is None:
                out[sl] = tr.reshape(out[sl].shape)
            else:
                out[sl, r] = tr

    def apply_S(self, g):
        g = self.check(g)
        out = np.zeros(g.shape, dtype=complex)
        g2 = g if g.ndim == 2 else g[:, None]
        o2 = out if out.ndim == 2 else out[:, None]
        for s in self.lat.subs:
            self._write(o2, self.scatter_one(s, g2))
        return out

    def apply_A(self, g):
        """(I - S) g (interface_system.py:144-146)."""
        g = self.check(g)
        return g.copy() - self.apply_S(g)

    def restricted(self, g, src_groups, tgt_groups):
        """V_T S V_Src^T g (interface_system.py:148-162)."""
        g = self.check(g)
        src, tgt = set(src_groups), set(tgt_groups)
        out = np.zeros(g.shape, dtype=complex)
        g2 = g if g.ndim == 2 else g[:, None]
        o2 = out if out.ndim == 2 else out[:, None]
        for s in self.lat.subs:
            if s[0] + s[1] in src:
                self._write(o2, self.scatter_one(s, g2, tgt))
        return out

    # ---- right-hand side (interface_system.py:98-113)
    def liftings(self):
        res = {}
        for s in self.lat.subs:
            if self.backend == "superlu" or s == self.home:
                op = self.ops[s] if self.backend == "superlu" else Subdomain(self.prob, self.lat, s)
                res[s] = op.lifting()
            else:
                res[s] = (np.zeros(self.n * self.n, complex), {f: np.zeros(self.n, complex) for f, _ in self.lat.faces[s]})
        return res

    def rhs(self, lifts=None):
        lifts = self.liftings() if lifts is None else lifts
        b = np.zeros(self.size, dtype=complex)
        for s in self.lat.subs:
            _, tr = lifts[s]
            for f, j in self.lat.faces[s]:
                b[self.block(self.lat.m_index(j, s))] = tr[f]
        return b

    def dense_S(self):
        if self.size > DENSE_GUARD:
            raise ValueError(f"dense guard exceeded: {self.size} > {DENSE_GUARD}")
        return self.apply_S(np.eye(self.size, dtype=complex))
