"""CPU: the drop-in boundary accepts the reference's OWN objects.

`GpuInterfaceSystem(spec, partition, imp=None, workers=1)` mirrors
`InterfaceSystem.__init__` (interface_system.py:73-89).  Here the arguments are
`helmsweep.discretization.ProblemSpec` / `helmsweep.indexing.Partition` /
`ImpedanceSpec` instances built by the real reference (imported from
/root/reference in the build container; skipped where it is absent, e.g. on
the GPU box).  A plan-only system (device=-1: the host side of the boundary,
no GPU) is built from them and checked against the reference: vector layout,
m-order tables, operator metadata (faces, interface neighbours, scatterer
cells), lifting data, windows and the sweep schedule.
"""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
if not os.path.isdir(REF):
    pytest.skip("reference package not present (build container only)", allow_module_level=True)
sys.path.insert(0, REF)

from helmsweep import discretization as rd  # noqa: E402
from helmsweep import indexing as ri  # noqa: E402
from helmsweep import interface_system as ris  # noqa: E402

from paper_2209_10886_b200.configs import CONFIGS, small_case  # noqa: E402
from paper_2209_10886_b200.discretization import lifting_data  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

CASES = {"cfg1": CONFIGS[1], "small_3x2": small_case(3, 2, 12), "cfg2": CONFIGS[2]}


def ref_objects(c):
    spec = rd.ProblemSpec(kappa=c["kappa"], cells_per_side=c["n"], subdomain_side=c["side"],
                          scatterer=rd.Scatterer(tuple(c["center"]), c["radius"]),
                          incident_direction=(float(np.cos(c["angle"])), float(np.sin(c["angle"]))))
    return spec, ri.Partition(c["n1"], c["n2"])


@pytest.mark.parametrize("name", list(CASES))
def test_plan_only_system_from_reference_objects(name):
    c = CASES[name]
    spec, part = ref_objects(c)
    imp = rd.ImpedanceSpec.for_problem(spec)
    gs = GpuInterfaceSystem(spec, part, imp, workers=1, device=-1)
    rs = ris.InterfaceSystem(spec, part, imp) if c["n"] <= 32 else None
    # layout (interface_system.py:30-62)
    assert gs.layout.size == ris.TraceLayout(part, spec.cells_per_side).size
    assert gs.spec is spec and gs.partition is part and gs.imp is imp
    # m-order: the native plan's pair table equals the reference's (indexing.py:114-148)
    tab = gs.ctx.pairs()
    want = np.array([[p.owner.i1, p.owner.i2, p.neighbor.i1, p.neighbor.i2] for p in part.pairs])
    assert np.array_equal(np.asarray(tab).reshape(-1, 4), want)
    for m, p in enumerate(part.pairs, start=1):
        assert gs.layout.block_of(p.owner, p.neighbor) == slice((m - 1) * spec.cells_per_side, m * spec.cells_per_side)
    # operator metadata (discretization.py:126-166) against the reference operators
    if rs is not None:
        for i, op in rs.operators.items():
            mine = gs.operators[i]
            assert dict(mine.interface_faces) == dict(op.interface_faces)
            assert np.array_equal(np.sort(mine.dirichlet_cells), np.sort(op.dirichlet_cells))
            for f in ("west", "east", "south", "north"):
                assert np.array_equal(mine.faces[f], op.faces[f])
    # lifting data: -u_inc at the reference's scatterer cells (discretization.py:315-332)
    home, data = lifting_data(spec, part)
    assert tuple(home) == tuple(rd.scatterer_subdomain(spec, part))
    if rs is not None:
        op = rs.operators[ri.MultiIndex(*home)]
        x, y = op.cell_x.ravel()[op.dirichlet_cells], op.cell_y.ravel()[op.dirichlet_cells]
        assert np.array_equal(data[:, 0], -spec.incident_wave(x, y))
    # windows (indexing.py:158-179) and the schedule built from them
    for kind in ("lower", "upper"):
        w = [(x.lo, x.hi) for x in ri.build_windows(part, kind)]
        from paper_2209_10886_b200.indexing import window_ranges
        assert window_ranges(part.n1, part.n2, kind, None) == w
    recs = gs.step_schedule("bsp")
    nf = max(hi - lo for lo, hi in [(x.lo, x.hi) for x in ri.build_windows(part, "lower")])
    assert sum(1 for r in recs if r[1] == "forward") == nf
    for _, ph, subs in recs:
        assert all(isinstance(s, tuple) and len(s) == 2 for s in subs)
    # every numerical entry point needs the GPU: a plan-only system refuses loudly
    with pytest.raises(ValueError, match="plan-only"):
        gs.apply_interface_operator(np.zeros(gs.layout.size, complex))


def test_sp_schedule_counts_from_reference_partition():
    """Table 1's structural step counts from a reference Partition."""
    for n2, ns_sp in [(5, 16), (10, 26), (15, 36), (20, 46)]:
        c = dict(small_case(5, n2, 8))
        spec, part = ref_objects(c)
        gs = GpuInterfaceSystem(spec, part, device=-1, sweep=SweepConfig(kind="sp"))
        assert len(gs.step_schedule("sp")) == ns_sp
        assert len(gs.step_schedule("bsp")) == 10
