"""CPU: the C-ABI library loads, exports every symbol include/hsb200.h declares,
and its host plan (m-order, windows, step schedule, row-band exchange) agrees
with the oracle.  No kernels run here (plan-only contexts, device -1)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2209_10886_b200 import native
from paper_2209_10886_b200.indexing import Partition, build_windows, window_ranges
from paper_2209_10886_b200.interface_system import schedule_records, SweepConfig

from oracle.lattice import Lattice, windows
from oracle.sweeps import SchedulePlan, step_schedule

LATTICES = [(1, 1), (1, 4), (2, 2), (3, 3), (4, 4), (5, 5), (5, 10), (6, 3), (8, 8), (16, 16), (32, 16)]


def test_every_header_symbol_is_exported():
    with open(os.path.join(ROOT, "include", "hsb200.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(hs_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(native.lib, name), name
    assert declared == set(native.EXPORTS)
    assert native.version().startswith("hsb200")


def test_errors_map_to_python_exceptions():
    with pytest.raises(ValueError):
        native.Context(-1, 0, 4, 8, 0.1, 1.0, 1j)
    with pytest.raises(ValueError):
        native.Context(-1, 2, 2, 8, 0.1, 1.0, 1.0)  # real impedance (discretization.py:96-98)
    with pytest.raises(ValueError):
        native.Context(-1, 2, 2, 3, 0.1, 1.0, 1j)   # cells_per_side < 4
    ctx = native.Context(-1, 2, 2, 8, 0.1, 1.0, 1j)
    with pytest.raises(ValueError):
        ctx.call("hs_factor")  # plan-only context cannot run kernels


@pytest.mark.parametrize("n1,n2", LATTICES)
def test_pairs_match_oracle(n1, n2):
    lat = Lattice(n1, n2)
    ctx = native.Context(-1, n1, n2, 8, 0.1, 1.0, 1j)
    want = np.array([[o[0], o[1], j[0], j[1]] for o, j in lat.pairs], dtype=np.int32).reshape(-1, 4)
    assert np.array_equal(ctx.pairs(), want)
    assert ctx.L == lat.n_pairs * 8 and ctx.nsub == n1 * n2 and ctx.ngroups == n1 + n2 - 1
    part = Partition(n1, n2)
    assert [tuple(map(tuple, p)) for p in part.pairs] == [tuple(p) for p in lat.pairs]
    assert part.n_interfaces == lat.n_interfaces and part.n_groups == lat.n_groups
    for k, p in enumerate(part.pairs, start=1):
        assert part.m_index(p) == k and part.m_invert(k) == p


@pytest.mark.parametrize("n1,n2", LATTICES)
@pytest.mark.parametrize("p", [None, 1, 2, 3, 4, 8])
def test_windows_match_oracle(n1, n2, p):
    for kind in ("lower", "upper"):
        assert window_ranges(n1, n2, kind, p) == windows(n1, n2, kind, p)
    if p is None:
        part = Partition(n1, n2)
        assert [(w.lo, w.hi) for w in build_windows(part, "lower")] == windows(n1, n2, "lower")


@pytest.mark.parametrize("n1,n2", [(2, 2), (3, 3), (5, 5), (5, 10), (1, 4), (8, 8), (16, 16), (32, 16)])
@pytest.mark.parametrize("kind,p", [("sp", None), ("bsp", None), ("bsp", 1), ("bsp", 4), ("bsp", 8)])
def test_schedule_matches_oracle(n1, n2, kind, p):
    lat = Lattice(n1, n2)
    part = Partition(n1, n2)
    ctx = native.Context(-1, n1, n2, 8, 0.1, 1.0, 1j)
    cfg = SweepConfig(kind=kind, blocks=p)
    for k, kd in ((0, "lower"), (1, "upper")):
        w = window_ranges(n1, n2, kd, p)
        lo, hi = native.i32([a for a, _ in w]), native.i32([b for _, b in w])
        ctx.call("hs_set_windows", k, native.iptr(lo), native.iptr(hi), len(w))
    got = schedule_records(ctx, part, kind, cfg)
    want = step_schedule(SchedulePlan(lat, kind, blocks=p))
    assert [(t, ph, sorted(map(tuple, s))) for t, ph, s in got] == [(t, ph, sorted(s)) for t, ph, s in want]


@pytest.mark.parametrize("n1,n2,G", [(4, 4, 2), (8, 8, 2), (8, 8, 4), (16, 16, 8), (32, 16, 8), (5, 7, 3)])
def test_row_band_exchange_plan(n1, n2, G):
    """Every output block that crosses a band edge is sent exactly once, by the
    band of the solving subdomain to the band that owns it, and the receiver's
    list matches the sender's list slot by slot."""
    lat = Lattice(n1, n2)
    ctxs = [native.Context(-1, n1, n2, 8, 0.1, 1.0, 1j, rank=r, nranks=G) for r in range(G)]
    owner = ctxs[0].block_owner()
    rows = [lat.pairs[m][0][1] for m in range(lat.n_pairs)]
    # bands are contiguous, balanced row ranges
    for m in range(lat.n_pairs):
        assert owner[m] == min(r for r in range(G) if rows[m] < 1 + sum(n2 // G + (i < n2 % G) for i in range(r + 1)))
    for kind in (0, 1, 2):
        for r in range(G):
            for peer in (r - 1, r + 1):
                if not 0 <= peer < G:
                    continue
                sent = ctxs[r].exchange_plan(kind, peer, recv=False)
                got = ctxs[peer].exchange_plan(kind, r, recv=True)
                assert np.array_equal(sent, got)
                for t, blk, slot in sent:
                    assert owner[blk] == peer
                    writer = lat.pairs[blk][1]  # block m(j, i) is written by i
                    assert ctxs[0].block_owner()[lat.first_block[writer] - 1] == r
                # forward steps only push north, backward only south
                if kind == 0:
                    assert peer == r + 1 or len(sent) == 0
                if kind == 1:
                    assert peer == r - 1 or len(sent) == 0
        # completeness: the full step moves every block whose writer and owner differ
        if kind == 2:
            crossing = {m for m in range(lat.n_pairs)
                        if owner[m] != ctxs[0].block_owner()[lat.first_block[lat.pairs[m][1]] - 1]}
            moved = set()
            for r in range(G):
                for peer in (r - 1, r + 1):
                    if 0 <= peer < G:
                        moved |= {int(b) for _, b, _ in ctxs[r].exchange_plan(2, peer)}
            assert moved == crossing


def test_step_records_read_write_disjoint():
    """every sweep step record's written blocks are distinct and
    disjoint from the blocks it reads in z -- checked by the native plan for
    every lattice / block count the schedules are built for (hs_schedule fails
    on a violation), and a violation is caught: overlapping windows make a
    subdomain write into a slab another solve of the same step reads."""
    import ctypes as C
    from paper_2209_10886_b200 import native
    from paper_2209_10886_b200.indexing import window_ranges
    for n1, n2 in [(4, 4), (8, 8), (5, 10), (6, 3), (16, 16), (32, 16), (1, 5), (7, 2)]:
        for p in (None, 1, 2, 3, 4, 8):
            ctx = native.Context(-1, n1, n2, 8, 0.1, 2.0, 2.0j, 0, 1)
            for k, kind in ((0, "lower"), (1, "upper")):
                w = window_ranges(n1, n2, kind, p)
                lo, hi = native.i32([a for a, _ in w]), native.i32([b for _, b in w])
                ctx.call("hs_set_windows", k, native.iptr(lo), native.iptr(hi), len(w))
            ctx.schedule(native.HS_PC_BSP)
            ctx.schedule(native.HS_PC_SP)
    ctx = native.Context(-1, 5, 5, 8, 0.1, 2.0, 2.0j, 0, 1)
    lo, hi = native.i32([2, 3]), native.i32([5, 6])
    ctx.call("hs_set_windows", 0, native.iptr(lo), native.iptr(hi), 2)
    with pytest.raises(ValueError, match="unsafe sweep"):
        ctx.schedule(native.HS_PC_BSP)
