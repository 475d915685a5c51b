"""Lattice numbering with the reference API (indexing.py:19-179), backed by the
native plan of libhsb200 (the same tables the GPU step kernels use).

`Partition(n1, n2)` exposes the reference attributes (`subdomains`,
`neighbors`, `pairs`, `n_interfaces`, `n_groups`, `groups`, `m_index`,
`m_invert`, `group_span`).  `build_windows(partition, kind, blocks=None)`
extends the reference rule with the block-count generalisation of SURVEY.md §8d.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple

from . import native


class MultiIndex(NamedTuple):
    i1: int
    i2: int

    @property
    def group(self) -> int:
        return self.i1 + self.i2


class DirectedPair(NamedTuple):
    owner: MultiIndex
    neighbor: MultiIndex


def _mkey(a) -> tuple[int, int]:
    return (a[0] + a[1], a[0])


def lex_less_multi(a, b) -> bool:
    """indexing.py:39-41: first |i|_1, then the column."""
    return _mkey(a) < _mkey(b)


def lex_less_pair(p, q) -> bool:
    """indexing.py:44-46: owner first, then neighbour."""
    return (_mkey(p[0]), _mkey(p[1])) < (_mkey(q[0]), _mkey(q[1]))


@dataclass(frozen=True)
class GroupWindow:
    kind: str
    block_index: int
    lo: int
    hi: int

    @property
    def groups(self) -> range:
        return range(self.lo, self.hi + 1)

    def __len__(self) -> int:
        return self.hi - self.lo + 1


class Partition:
    """N1 x N2 checkerboard with m-ordered directed pairs (indexing.py:79-151)."""

    def __init__(self, n1: int, n2: int):
        if n1 < 1 or n2 < 1:
            raise ValueError(f"partition dimensions must be positive, got {n1}x{n2}")
        self.n1, self.n2 = int(n1), int(n2)
        plan = native.Context(-1, n1, n2, 4, 1.0, 1.0, 1j)
        tab = plan.pairs()
        self.pairs = tuple(DirectedPair(MultiIndex(int(a), int(b)), MultiIndex(int(c), int(d))) for a, b, c, d in tab)
        self.subdomains = tuple(sorted((MultiIndex(a, b) for b in range(1, n2 + 1) for a in range(1, n1 + 1)), key=_mkey))
        nb = {s: [] for s in self.subdomains}
        for p in self.pairs:
            nb[p.owner].append(p.neighbor)
        self.neighbors = {s: tuple(v) for s, v in nb.items()}
        self._ordinal = {p: k for k, p in enumerate(self.pairs, start=1)}
        self.n_interfaces = 2 * self.n1 * self.n2 - self.n1 - self.n2
        self.n_groups = self.n1 + self.n2 - 1
        self.groups: dict[int, tuple[MultiIndex, ...]] = {}
        for s in self.subdomains:
            self.groups[s.group] = self.groups.get(s.group, ()) + (s,)

    @property
    def n_subdomains(self) -> int:
        return self.n1 * self.n2

    @property
    def group_span(self) -> range:
        return range(2, self.n_groups + 2)

    def m_index(self, pair) -> int:
        try:
            key = DirectedPair(MultiIndex(*pair[0]), MultiIndex(*pair[1]))
            return self._ordinal[key]
        except (KeyError, TypeError):
            raise ValueError(f"{pair!r} is not a directed interface of this {self.n1}x{self.n2} partition") from None

    def m_invert(self, k: int) -> DirectedPair:
        if not 1 <= k <= len(self.pairs):
            raise ValueError(f"ordinal {k} out of range 1..{len(self.pairs)}")
        return self.pairs[k - 1]

    def __repr__(self) -> str:
        return f"Partition({self.n1}x{self.n2}, N_e={self.n_interfaces}, N_g={self.n_groups})"


def build_partition(n1: int, n2: int) -> Partition:
    return Partition(n1, n2)


def window_ranges(n1: int, n2: int, kind: str, blocks: int | None = None) -> list[tuple[int, int]]:
    """Inclusive (lo, hi) group windows.  blocks None / the reference count ->
    indexing.py:158-179; otherwise the SURVEY.md §8d rules (ii)/(iii)."""
    if kind not in ("lower", "upper"):
        raise ValueError(f"window kind must be 'lower' or 'upper', got {kind!r}")
    ng = n1 + n2 - 1
    steps = ng - 1
    if steps <= 0:
        return []
    p_ref = math.ceil(steps / n1)
    if blocks is None or blocks == p_ref:
        lens = None
        out = []
        for b in range(1, p_ref + 1):
            if kind == "lower":
                lo, hi = 2 + (b - 1) * n1, 2 + b * n1
            else:
                lo, hi = ng + 1 - b * n1, ng + 1 - (b - 1) * n1
            out.append((max(lo, 2), min(hi, ng + 1)))
        return out
    if blocks < 1:
        raise ValueError("block count must be >= 1")
    p = min(int(blocks), steps)
    w = math.ceil(steps / p)
    if math.ceil(steps / w) == p:
        lens = [w] * (steps // w) + ([steps % w] if steps % w else [])
    else:
        base, extra = divmod(steps, p)
        lens = [base + 1] * extra + [base] * (p - extra)
    lower, lo = [], 2
    for ln in lens:
        lower.append((lo, lo + ln))
        lo += ln
    if kind == "lower":
        return lower
    return [(ng + 3 - hi, ng + 3 - lo) for lo, hi in lower]


def build_windows(partition: Partition, kind: str, blocks: int | None = None) -> list[GroupWindow]:
    return [GroupWindow(kind, b, lo, hi)
            for b, (lo, hi) in enumerate(window_ranges(partition.n1, partition.n2, kind, blocks), start=1)]
