"""Process-parallel driver of the REAL reference InterfaceSystem (build container only).

Two harness-level changes make configs 3 and 5 affordable with the reference's
own arithmetic; neither modifies a reference file:

* Shared factors.  `_assemble_grid` (discretization.py:221-256) uses the same
  ghost ratio s/d on all four faces (:224-229), so every subdomain without
  scatterer cells has a bitwise identical matrix.  `shared_splu()` replaces the
  module-level `splu` that `LocalOperator.__init__` calls (discretization.py:172)
  by a cache keyed on the exact CSC arrays (data, indices, indptr, shape): a
  second identical matrix gets the SuperLU object the first one produced.
  SuperLU's factorisation is deterministic and `solve` is read-only on it
  (discretization.py:119-123, 183-184), so every solve is bit-for-bit the one
  the unshared reference would do.  cfg5 then needs 2 factors (~200 MB)
  instead of 512 (~52 GB).  `make_golden.py --check-cfg3` proves it against
  the committed cfg3 golden (generated with one factor per subdomain).

* Process parallelism.  `restricted_apply` / `apply_scattering`
  (interface_system.py:135-162) run one independent `_scatter_one` per
  subdomain and assign each output block exactly once (:68-71).  `ParAdapter`
  runs the reference's own `_scatter_one` for disjoint subdomain chunks in
  forked worker processes and assigns the returned blocks into a zeroed
  vector, exactly as the reference loop does; the result is bitwise the
  serial reference result for any worker count (the reference's own
  determinism contract).  The input vector travels through
  one shared-memory buffer.
"""

from __future__ import annotations

import hashlib
import multiprocessing as mp
import os
from contextlib import contextmanager
from multiprocessing import shared_memory

import numpy as np

_SYS = None  # the reference InterfaceSystem, inherited by forked workers
_SHM = None
_L = 0


@contextmanager
def shared_splu(ref_disc):
    orig = ref_disc.splu
    cache = {}
    stats = {"factor": 0, "reuse": 0}

    def cached(A):
        A = A.tocsc()
        h = hashlib.sha256()
        for arr in (A.data, A.indices, A.indptr, np.asarray(A.shape)):
            h.update(np.ascontiguousarray(arr).tobytes())
        key = h.hexdigest()
        if key not in cache:
            cache[key] = orig(A)
            stats["factor"] += 1
        else:
            stats["reuse"] += 1
        return cache[key]

    ref_disc.splu = cached
    try:
        yield stats
    finally:
        ref_disc.splu = orig


def _work(args):
    subs, targets = args
    g = np.ndarray((_L,), dtype=complex, buffer=_SHM.buf)
    out = []
    for i in subs:
        for sl, trace in _SYS._scatter_one(i, g, targets):
            out.append((sl.start, sl.stop, trace))
    return out


class ParAdapter:
    """Oracle `Interface` API (restricted / apply_A) over the reference system,
    evaluated by `workers` forked processes."""

    def __init__(self, system, lat, workers=None):
        global _SYS, _SHM, _L
        self.sys = system
        self.lat = lat
        self.size = system.layout.size
        self.n = system.layout.n
        _SYS = system
        _L = self.size
        _SHM = shared_memory.SharedMemory(create=True, size=16 * self.size)
        self.shm = _SHM
        self.g = np.ndarray((self.size,), dtype=complex, buffer=_SHM.buf)
        self.workers = workers or os.cpu_count()
        self.pool = mp.get_context("fork").Pool(self.workers)
        self.subs = list(system.partition.subdomains)

    def close(self):
        self.pool.close()
        self.pool.join()
        self.shm.close()
        self.shm.unlink()

    def _run(self, g, solves, targets):
        g = self.sys.layout.check(g)
        self.g[:] = g
        out = self.sys.layout.zeros()
        chunks = [solves[w::self.workers] for w in range(self.workers)]
        for writes in self.pool.map(_work, [(c, targets) for c in chunks if c]):
            for a, b, trace in writes:
                out[a:b] = trace
        return out

    # reference: interface_system.py:135-142
    def apply_S(self, g):
        return self._run(g, self.subs, None)

    # reference: interface_system.py:144-146
    def _apply_A1(self, g):
        return self.sys.layout.check(g).copy() - self.apply_S(g)

    # reference: interface_system.py:148-162
    def _restricted1(self, g, src, tgt):
        src, tgt = set(src), set(tgt)
        return self._run(g, [i for i in self.subs if i.group in src], tgt)

    def restricted(self, g, src, tgt):
        g = np.asarray(g)
        if g.ndim == 1:
            return self._restricted1(g, src, tgt)
        return np.stack([self._restricted1(g[:, r], src, tgt) for r in range(g.shape[1])], 1)

    def apply_A(self, g):
        g = np.asarray(g)
        if g.ndim == 1:
            return self._apply_A1(g)
        return np.stack([self._apply_A1(g[:, r]) for r in range(g.shape[1])], 1)
