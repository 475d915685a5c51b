"""Preconditioner entry points of SPEC.md:306-357 (not shipped by the reference)
as free functions over a GpuInterfaceSystem, plus the StepTrace format."""

from __future__ import annotations

from .interface_system import GpuInterfaceSystem, SweepConfig


def forward_sweep(system: GpuInterfaceSystem, r):
    return system.forward_sweep(r)


def backward_sweep(system: GpuInterfaceSystem, r):
    return system.backward_sweep(r)


def sgs_apply(system: GpuInterfaceSystem, r):
    return system.sgs_apply(r)


def bj_half_apply(system: GpuInterfaceSystem, r, direction: str):
    return system.bj_half_apply(r, direction)


def bsp_apply(system: GpuInterfaceSystem, b):
    return system.bsp_apply(b)


def step_schedule(config: SweepConfig, system: GpuInterfaceSystem):
    """Schedule of `config`; the system's own configuration
    is restored afterwards."""
    if config.kind == "none":
        return []
    with system.using(config):
        return system.step_schedule(config.kind)


def steps_per_apply(config: SweepConfig, system: GpuInterfaceSystem) -> int:
    return len(step_schedule(config, system))


def format_trace(records) -> str:
    """`step=<t> phase=<...> solves=(i1,i2);...` lines."""
    return "".join(f"step={t} phase={ph} solves=" + ";".join(f"({a},{b})" for a, b in subs) + "\n"
                   for t, ph, subs in records)


def make_preconditioner(system: GpuInterfaceSystem, config: SweepConfig):
    """apply_M for krylov.gmres; carries its system, kind and configuration
    for the device fast path.  Each call runs under the preconditioner's own
    configuration (the system's current one is restored afterwards), so
    preconditioners built for different configurations coexist."""
    config = SweepConfig(**vars(config))  # a snapshot: later edits of the caller's object do not leak in

    class _M:
        kind = config.kind
        owner = system
        sweep = config

        def __call__(self, r):
            with system.using(config):
                return system.precondition(r, config.kind)

    return _M()
