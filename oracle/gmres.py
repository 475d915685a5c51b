"""Full right-preconditioned GMRES with MGS Arnoldi and Givens rotations
(oracle restatement of SPEC.md:384-424; the reference ships no krylov module).

Conventions fixed here and mirrored by the GPU (they decide iteration counts):
  * x0 = 0, beta = ||b||, b = 0 -> x = 0 after 0 iterations;
  * right preconditioning: A M w = b, x = M (V y);
  * modified Gram-Schmidt in j = 0..k order, h_jk = <v_j, w> = v_j^H w;
  * complex Givens with real cosine: c = |a|/rho, s = (a/|a|) conj(b)/rho
    (c = 0, s = 1 when a = 0);
  * stop at the first k with |g_{k+1}| / beta <= tol (internal residual);
    history[0] = 1 and history[k] = |g_k|/beta (iterations+1 rows);
  * breakdown when h_{k+1,k} <= 16 eps ||A M v_k|| before orthogonalisation,
    reported separately from non-convergence.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

EPS = np.finfo(float).eps


@dataclass
class GmresOut:
    x: np.ndarray
    iterations: int
    converged: bool
    history: list = field(default_factory=list)
    breakdown: bool = False
    basis: list = field(default_factory=list)  # the Arnoldi vectors v_0 .. v_{iterations-1}


def givens(a: complex, b: float):
    if a == 0:
        return 0.0, 1.0 + 0j
    rho = np.hypot(abs(a), abs(b))
    return abs(a) / rho, (a / abs(a)) * np.conj(b) / rho


def gmres(apply_A, apply_M, b, tol: float = 1e-6, maxit: int = 200) -> GmresOut:
    b = np.asarray(b, dtype=complex)
    beta = float(np.linalg.norm(b))
    if beta == 0.0:
        return GmresOut(np.zeros_like(b), 0, True, [])
    V = [b / beta]
    H = np.zeros((maxit + 1, maxit), dtype=complex)
    cs = np.zeros(maxit)
    sn = np.zeros(maxit, dtype=complex)
    g = np.zeros(maxit + 1, dtype=complex)
    g[0] = beta
    hist = [1.0]
    k_done, conv, brk = 0, False, False
    for k in range(maxit):
        z = apply_M(V[k]) if apply_M is not None else V[k]
        w = np.array(apply_A(z), dtype=complex)
        wnorm0 = np.linalg.norm(w)
        for j in range(k + 1):
            H[j, k] = np.vdot(V[j], w)
            w = w - H[j, k] * V[j]
        hn = np.linalg.norm(w)
        H[k + 1, k] = hn
        for j in range(k):
            t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
            H[j + 1, k] = -np.conj(sn[j]) * H[j, k] + cs[j] * H[j + 1, k]
            H[j, k] = t
        c, s = givens(H[k, k], H[k + 1, k].real)
        cs[k], sn[k] = c, s
        H[k, k] = c * H[k, k] + s * H[k + 1, k]
        H[k + 1, k] = 0.0
        g[k + 1] = -np.conj(s) * g[k]
        g[k] = c * g[k]
        res = abs(g[k + 1]) / beta
        hist.append(float(res))
        k_done = k + 1
        if res <= tol:
            conv = True
            break
        if hn <= 16 * EPS * wnorm0:
            brk = True
            break
        V.append(w / hn)
    m = k_done
    y = np.zeros(m, dtype=complex)
    for i in range(m - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1:m] @ y[i + 1:m]) / H[i, i]
    u = sum(y[i] * V[i] for i in range(m))
    x = apply_M(u) if apply_M is not None else u
    return GmresOut(np.asarray(x), m, conv, hist, brk, V[:m])
