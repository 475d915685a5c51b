"""`gmres(apply_A, apply_M, b, opts)` on the device.

The spec's signature takes operator callables; the GPU fast path applies when
`apply_A` is a GpuInterfaceSystem's `apply_interface_operator` and `apply_M`
is None or a preconditioner built by `preconditioner.make_preconditioner` /
one of the system's preconditioner methods.  Anything else is rejected
(there is no host GMRES in the product; the CPU restatement lives in
oracle/gmres.py as test infrastructure).
"""

from __future__ import annotations

from .interface_system import GmresOptions, GmresResult, GpuInterfaceSystem


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


def gmres(apply_A, apply_M, b, opts: GmresOptions | None = None) -> GmresResult:
    opts = opts or GmresOptions()
    system = _system_of(apply_A)
    if system is None:
        raise TypeError("gmres: apply_A must be GpuInterfaceSystem.apply_interface_operator")
    kind = _kind_of(apply_M, system)
    if kind is None:
        raise TypeError("gmres: apply_M must be None or a preconditioner of the same GpuInterfaceSystem")
    sweep = getattr(apply_M, "sweep", None) if getattr(apply_M, "owner", None) is system else None
    if sweep is None:
        return system.gmres(b, kind=kind, tol=opts.tol, maxit=opts.maxit)
    with system.using(sweep):  # the preconditioner's own windows / seams
        return system.gmres(b, kind=kind, tol=opts.tol, maxit=opts.maxit)
