"""`gmres(apply_A, apply_M, b, opts)` on the device.

The spec's signature takes operator callables.  The fast path applies when
`apply_A` is a GpuInterfaceSystem's `apply_interface_operator` and `apply_M`
is None or a preconditioner built by `preconditioner.make_preconditioner` /
one of the system's preconditioner methods: the whole solve is the library's
hs_gmres (fused A M v launches, one Arnoldi kernel per iteration).  Any other
pair of linear callables runs the same algorithm -- right preconditioning,
MGS Arnoldi, complex Givens with a real cosine, the internal-residual stop,
the 16 eps breakdown test (oracle/gmres.py header: the conventions that
decide iteration counts) -- with the Krylov basis on the GPU (torch CUDA
tensors); the callables receive and return vectors of the kind of b (numpy
or torch).  There is no host GMRES in the product.
"""

from __future__ import annotations

import time

import numpy as np

from .interface_system import GmresOptions, GmresResult, GpuInterfaceSystem

_EPS = float(np.finfo(float).eps)


def _system_of(apply_A) -> GpuInterfaceSystem | None:
    owner = getattr(apply_A, "__self__", None)
    if isinstance(owner, GpuInterfaceSystem) and apply_A.__func__ is GpuInterfaceSystem.apply_interface_operator:
        return owner
    return None


def _kind_of(apply_M, system) -> str | None:
    if apply_M is None:
        return "none"
    if getattr(apply_M, "owner", None) is system:
        return apply_M.kind
    owner = getattr(apply_M, "__self__", None)
    if owner is system:
        f = apply_M.__func__
        if f is GpuInterfaceSystem.bsp_apply:
            return "bsp"
        if f is GpuInterfaceSystem.sgs_apply:
            return "sp"
    return None


def _generic(apply_A, apply_M, b, tol: float, maxit: int) -> GmresResult:
    """SPEC.md:399-407 for arbitrary linear callables; the basis, the
    orthogonalisation and the update live on the GPU."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("gmres: the generic path needs a CUDA device (no host GMRES in the product)")
    t0 = time.perf_counter()
    is_torch = isinstance(b, torch.Tensor)
    dev = torch.device("cuda")
    bt = (b.to(dev) if is_torch else torch.from_numpy(np.ascontiguousarray(b)).to(dev)).to(torch.complex128).reshape(-1)

    def call(f, v):  # v: device tensor -> device tensor, through the caller's vector kind
        out = f(v if is_torch else v.cpu().numpy())
        out = out if isinstance(out, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(out))
        return out.to(dev).to(torch.complex128).reshape(-1)

    def wrap(x):
        return x if is_torch else x.cpu().numpy()

    beta = float(torch.linalg.vector_norm(bt))
    if beta == 0.0:  # b = 0 -> x = 0 after 0 iterations
        return GmresResult(wrap(torch.zeros_like(bt)), [], 0, True, time.perf_counter() - t0)
    V = [bt / beta]
    H = np.zeros((maxit + 1, maxit), dtype=complex)
    cs = np.zeros(maxit)
    sn = np.zeros(maxit, dtype=complex)
    g = np.zeros(maxit + 1, dtype=complex)
    g[0] = beta
    hist = [1.0]
    k_done, conv = 0, False
    for k in range(maxit):
        z = call(apply_M, V[k]) if apply_M is not None else V[k]
        w = call(apply_A, z)
        wnorm0 = float(torch.linalg.vector_norm(w))
        for j in range(k + 1):  # modified Gram-Schmidt, j = 0..k
            h = torch.vdot(V[j], w)
            H[j, k] = complex(h)
            w = w - h * V[j]
        hn = float(torch.linalg.vector_norm(w))
        H[k + 1, k] = hn
        for j in range(k):
            t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
            H[j + 1, k] = -np.conj(sn[j]) * H[j, k] + cs[j] * H[j + 1, k]
            H[j, k] = t
        a, bb = H[k, k], H[k + 1, k].real
        if a == 0:
            c, s = 0.0, 1.0 + 0j
        else:
            rho = np.hypot(abs(a), abs(bb))
            c, s = abs(a) / rho, (a / abs(a)) * np.conj(bb) / rho
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
        if hn <= 16 * _EPS * wnorm0:  # breakdown, reported as non-convergence with its history
            break
        V.append(w / hn)
    m = k_done
    y = np.zeros(m, dtype=complex)
    for i in range(m - 1, -1, -1):
        y[i] = (g[i] - H[i, i + 1:m] @ y[i + 1:m]) / H[i, i]
    u = torch.zeros_like(bt)
    for i in range(m):
        u = u + complex(y[i]) * V[i]
    x = call(apply_M, u) if apply_M is not None else u
    return GmresResult(wrap(x), hist, m, conv, time.perf_counter() - t0)


def gmres(apply_A, apply_M, b, opts: GmresOptions | None = None) -> GmresResult:
    opts = opts or GmresOptions()
    system = _system_of(apply_A)
    kind = _kind_of(apply_M, system) if system is not None else None
    if system is None or kind is None:
        # arbitrary linear callables: the same algorithm, basis on the GPU
        return _generic(apply_A, apply_M, b, opts.tol, opts.maxit)
    sweep = getattr(apply_M, "sweep", None) if getattr(apply_M, "owner", None) is system else None
    if sweep is None:
        return system.gmres(b, kind=kind, tol=opts.tol, maxit=opts.maxit)
    with system.using(sweep):  # the preconditioner's own windows / seams
        return system.gmres(b, kind=kind, tol=opts.tol, maxit=opts.maxit)
