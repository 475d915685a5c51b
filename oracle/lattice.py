"""Checkerboard lattice, directed-pair numbering and sweep windows (oracle).

Restates `/root/reference/pkg/src/helmsweep/indexing.py`:
  * multi-index order (|i|_1, i1)            -> indexing.py:39-54
  * subdomain list, neighbour sets D_i       -> indexing.py:100-112
  * directed pairs in m-order, m / m^-1      -> indexing.py:114-148
  * N_e, N_g, diagonal groups                -> indexing.py:119-126
  * block windows of the partial sweeps      -> indexing.py:158-179
plus the block-count generalisation of the windows agreed in SURVEY.md §8d
(rules (i)-(iii)); the reference has no block-count parameter
(SPEC.md:380 open question).
"""

from __future__ import annotations

import math

# Face order of one owner's blocks in m-order: W, S, N, E (the neighbour keys
# (|j|_1, j1) sort exactly like this, see indexing.py:111).
FACE_NAMES = ("west", "south", "north", "east")
FACE_STEP = ((-1, 0), (0, -1), (0, 1), (1, 0))


def _key(a):
    return (a[0] + a[1], a[0])


class Lattice:
    """N1 x N2 lattice with its m-ordered directed pairs (indexing.py:79-151)."""

    def __init__(self, n1: int, n2: int):
        if n1 < 1 or n2 < 1:
            raise ValueError(f"partition dimensions must be positive, got {n1}x{n2}")
        self.n1, self.n2 = n1, n2
        self.subs = sorted(((a, b) for a in range(1, n1 + 1) for b in range(1, n2 + 1)), key=_key)
        self.n_interfaces = 2 * n1 * n2 - n1 - n2
        self.n_groups = n1 + n2 - 1
        # faces[i] = [(face_index, neighbour)] in W,S,N,E order (= neighbour key order)
        self.faces = {}
        for s in self.subs:
            lst = []
            for f, (d1, d2) in enumerate(FACE_STEP):
                j = (s[0] + d1, s[1] + d2)
                if 1 <= j[0] <= n1 and 1 <= j[1] <= n2:
                    lst.append((f, j))
            self.faces[s] = lst
        # m-order: owners in multi-index order, then neighbours in key order
        self.pairs = []
        self.first_block = {}
        for s in self.subs:
            self.first_block[s] = len(self.pairs) + 1
            self.pairs.extend((s, j) for _, j in self.faces[s])
        self.m = {p: k for k, p in enumerate(self.pairs, start=1)}
        assert len(self.pairs) == 2 * self.n_interfaces
        self.groups = {}
        for s in self.subs:
            self.groups.setdefault(s[0] + s[1], []).append(s)

    @property
    def n_pairs(self) -> int:
        return len(self.pairs)

    def m_index(self, owner, neighbor) -> int:
        try:
            return self.m[(tuple(owner), tuple(neighbor))]
        except KeyError:
            raise ValueError(f"({owner}, {neighbor}) is not a directed interface") from None

    def block_group(self):
        """|owner|_1 of every block in m-order (length 2 N_e)."""
        return [o[0] + o[1] for o, _ in self.pairs]


def reference_windows(n1: int, n_groups: int, kind: str):
    """The reference rule p = ceil((N_g-1)/N1), windows of N1 group steps
    clipped to [2, N_g+1]; upper windows are the mirrored ranges
    (indexing.py:166-179).  Returns a list of (lo, hi)."""
    if kind not in ("lower", "upper"):
        raise ValueError(f"window kind must be 'lower' or 'upper', got {kind!r}")
    p = math.ceil((n_groups - 1) / n1)
    out = []
    for b in range(1, p + 1):
        if kind == "lower":
            lo, hi = 2 + (b - 1) * n1, 2 + b * n1
        else:
            lo, hi = (1 + n_groups) - b * n1, (1 + n_groups) - (b - 1) * n1
        out.append((max(lo, 2), min(hi, n_groups + 1)))
    return out


def windows(n1: int, n2: int, kind: str, p: int | None = None):
    """Window list shared by oracle and GPU:
    (i)   p absent or p == ceil((N_g-1)/N1): the reference rule;
    (ii)  else w = ceil((N_g-1)/p); if ceil((N_g-1)/w) == p use windows of w steps;
    (iii) else split the N_g-1 steps into p consecutive windows, the first
          (N_g-1) mod p of them one step longer.
    Upper windows mirror the lower ones via gamma -> N_g+3-gamma."""
    ng = n1 + n2 - 1
    steps = ng - 1
    if steps <= 0:
        return []
    p_ref = math.ceil(steps / n1)
    if p is None or p == p_ref:
        return reference_windows(n1, ng, kind)
    if p < 1:
        raise ValueError("block count must be >= 1")
    p = min(p, steps)
    w = math.ceil(steps / p)
    if math.ceil(steps / w) == p:
        lens = [w] * (steps // w) + ([steps % w] if steps % w else [])
    else:
        base, extra = divmod(steps, p)
        lens = [base + 1] * extra + [base] * (p - extra)
    lower = []
    lo = 2
    for ln in lens:
        lower.append((lo, lo + ln))
        lo += ln
    if kind == "lower":
        return lower
    if kind != "upper":
        raise ValueError(f"window kind must be 'lower' or 'upper', got {kind!r}")
    return [(ng + 3 - hi, ng + 3 - lo) for lo, hi in lower]
