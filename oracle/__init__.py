"""CPU oracle for the helmsweep hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference algorithm
(`/root/reference/pkg/src/helmsweep/*.py` for the shipped modules and
`/root/reference/SPEC.md:291-480` for the preconditioner / krylov / driver
modules the reference specifies but does not ship).  Every function cites the
reference file:line it restates.

Who may use it: `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py`, and only as the checker or the timed
CPU baseline.  The product package `paper_2209_10886_b200` never imports it;
its GPU path fails loudly when the CUDA library is missing.

Parity pinning: the restatement is checked against golden vectors produced by
importing the real reference in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`, tested by
`tests/test_oracle_golden.py`).  The sweeps/BSP/GMRES have no reference code,
so they are pinned against the SPEC.md known-answer examples and dense-matrix
identities (`tests/test_oracle_kat.py`).
"""

from .lattice import Lattice, windows, reference_windows
from .fd import Problem, Subdomain, mono_solve
from .interface import Interface
from .sweeps import Preconditioner, step_schedule
from .gmres import gmres, GmresOut
from .schur import schur_map, schur_maps_for

__all__ = [
    "Lattice", "windows", "reference_windows", "Problem", "Subdomain", "mono_solve",
    "Interface", "Preconditioner", "step_schedule", "gmres", "GmresOut",
    "schur_map", "schur_maps_for",
]
