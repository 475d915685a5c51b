"""Run artefacts of the SPEC front end: residuals.csv,
schedule.txt (StepTrace text), field.csv and report.txt, plus the
Table-1 style partition sweep.

Everything here is host-side formatting of a `driver.SolveReport`; the solve
itself runs on the GPU through `driver.solve_problem`.  Files are written with
fixed formatting (`%.17g`) so repeated runs of the same configuration are
byte-identical: the GPU path is deterministic (no atomics in any
reduction order) and wall times go to report.txt only when asked for.
"""

from __future__ import annotations

import os

import numpy as np

from .discretization import cell_centres


def format_schedule(recs) -> str:
    """StepTrace lines `step=<t> phase=<forward|backward|residual> solves=(i1,i2);...`."""
    return "".join(
        f"step={t} phase={ph} solves=" + ";".join(f"({int(s[0])},{int(s[1])})" for s in subs) + "\n"
        for t, ph, subs in recs)


def format_residuals(history) -> str:
    """`iteration,relative_residual`, one row per entry (iteration 0 = 1.0)."""
    return "iteration,relative_residual\n" + "".join(
        f"{k},{float(r):.17g}\n" for k, r in enumerate(history))


def format_field(spec, partition, field: np.ndarray) -> str:
    """`x,y,re,im` per cell centre of the stitched (N2 n) x (N1 n) field, y slow,
    with the `# kappa=... N1=... N2=... n=...` header."""
    n = spec.cells_per_side
    if field.shape != (partition.n2 * n, partition.n1 * n):
        raise ValueError(f"field shape {field.shape} does not match the {partition.n1}x{partition.n2} grid of n={n}")
    X = np.empty(field.shape)
    Y = np.empty(field.shape)
    for i in partition.subdomains:
        x, y = cell_centres(spec, i)
        sl = (slice((i[1] - 1) * n, i[1] * n), slice((i[0] - 1) * n, i[0] * n))
        X[sl], Y[sl] = x, y
    head = f"# kappa={spec.kappa:.17g} N1={partition.n1} N2={partition.n2} n={n}\n"
    rows = np.column_stack([X.ravel(), Y.ravel(), field.real.ravel(), field.imag.ravel()])
    return head + "".join(f"{a:.17g},{b:.17g},{c:.17g},{d:.17g}\n" for a, b, c, d in rows)


def format_report(report, spec, partition, kind: str, timings: bool = False) -> str:
    """report.txt: the SolveReport fields, one `key = value` per line."""
    lines = [
        f"N1 = {partition.n1}", f"N2 = {partition.n2}", f"cells_per_side = {spec.cells_per_side}",
        f"kappa = {spec.kappa:.17g}", f"precond = {kind}",
        f"converged = {str(bool(report.converged)).lower()}",
        f"iterations = {report.iterations}",
        f"steps_per_iteration = {report.steps_per_iteration}",
        f"total_sequential_steps = {report.total_sequential_steps}",
        f"final_relative_residual = {float(report.residual_history[-1]) if report.residual_history else 0.0:.17g}",
    ]
    if report.error_vs_mono is not None:
        lines += [f"error_vs_mono_max_rel = {report.error_vs_mono['max_rel']:.17g}",
                  f"error_vs_mono_l2_rel = {report.error_vs_mono['l2_rel']:.17g}"]
    if timings:
        lines += [f"wall_time = {report.wall_time:.6f}", f"setup_time = {report.setup_time:.6f}"]
    return "\n".join(lines) + "\n"


def write_artifacts(out_dir, report, spec, partition, kind: str, timings: bool = False) -> list[str]:
    """Write the four run artefacts; returns their paths."""
    os.makedirs(out_dir, exist_ok=True)
    files = {
        "residuals.csv": format_residuals(report.residual_history),
        "schedule.txt": format_schedule(report.schedule),
        "report.txt": format_report(report, spec, partition, kind, timings),
    }
    if report.field is not None:
        files["field.csv"] = format_field(spec, partition, report.field)
    paths = []
    for name, text in files.items():
        p = os.path.join(out_dir, name)
        with open(p, "w", newline="\n") as f:
            f.write(text)
        paths.append(p)
    return paths


TABLE_HEADER = "N1,N2,precond,ni,ns,t,converged,error\n"


def table_row(n1, n2, kind, report=None, error: str = "") -> str:
    """One Table-1 row: ni iterations, ns steps per iteration,
    t the GMRES-phase wall time; a failed row keeps its message in `error`."""
    if report is None:
        return f"{n1},{n2},{kind},,,,false,{error.replace(',', ';')}\n"
    return (f"{n1},{n2},{kind},{report.iterations},{report.steps_per_iteration},"
            f"{report.wall_time:.6f},{str(bool(report.converged)).lower()},\n")
