"""Process-parallel evaluation of the oracle's reference arithmetic -- TEST /
BASELINE INFRASTRUCTURE ONLY (bench.py's cpu_baseline and --impl reference legs).

The reference runs the subdomain solves of one application in a thread pool
(interface_system.py:91-96) that gives no speed-up (SciPy's SuperLU solve holds
the GIL), so the CPU baseline uses processes instead: forked
workers each run `Interface.scatter_one` (the restatement of
interface_system.py:115-133, bitwise equal to the reference, tests/
test_oracle_golden.py) for a disjoint chunk of the step's subdomains, and the
parent assigns the returned blocks exactly as `restricted_apply` /
`apply_scattering` do (interface_system.py:135-162).  Each output block has one
writer, so the result is bitwise the serial one for any worker count.  BLAS is
pinned to one thread per worker, so `workers` is the honest core count.
"""

from __future__ import annotations

import multiprocessing as mp
import os
from multiprocessing import shared_memory

import numpy as np

_ITF = None
_SHM = None
_L = 0


def _init():
    global _LIMIT
    try:
        from threadpoolctl import threadpool_limits
        _LIMIT = threadpool_limits(1)
    except Exception:  # pragma: no cover - threadpoolctl is in the image
        _LIMIT = None


def _work(args):
    subs, targets = args
    g = np.ndarray((_L, 1), dtype=complex, buffer=_SHM.buf)
    out = []
    solves = 0
    for s in subs:
        writes = _ITF.scatter_one(s, g, targets)
        solves += bool(writes)  # scatter_one returns no writes exactly when it skips the solve
        for sl, r, tr in writes:
            out.append((sl.start, sl.stop, np.asarray(tr).reshape(-1)))
    return solves, out


class ParInterface:
    """`Interface`-compatible restricted / apply_A / apply_S over a process pool
    (single right-hand side)."""

    def __init__(self, itf, workers: int | None = None):
        global _ITF, _SHM, _L
        self.itf = itf
        self.lat, self.n, self.size = itf.lat, itf.n, itf.size
        _ITF, _L = itf, itf.size
        _SHM = shared_memory.SharedMemory(create=True, size=16 * itf.size)
        self.shm = _SHM
        self.g = np.ndarray((itf.size,), dtype=complex, buffer=_SHM.buf)
        self.workers = max(1, int(workers or os.cpu_count() or 1))
        self.pool = mp.get_context("fork").Pool(self.workers, initializer=_init)
        self.solves = 0  # subdomain solves performed so far (the reference's unit of work)

    def close(self):
        self.pool.close()
        self.pool.join()
        self.shm.close()
        self.shm.unlink()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _run(self, g, solves, targets):
        g = self.itf.check(g)
        if g.ndim != 1:
            raise ValueError("ParInterface takes one right-hand side")
        self.g[:] = g
        out = np.zeros(self.size, dtype=complex)
        # round robin: every subdomain solve costs the same (one SuperLU solve of an n^2 system)
        chunks = [solves[w::self.workers] for w in range(self.workers)]
        for ns, writes in self.pool.map(_work, [(c, targets) for c in chunks if c]):
            self.solves += ns
            for a, b, tr in writes:
                out[a:b] = tr
        return out

    def apply_S(self, g):  # interface_system.py:135-142
        return self._run(g, list(self.lat.subs), None)

    def apply_A(self, g):  # interface_system.py:144-146
        return self.itf.check(g).copy() - self.apply_S(g)

    def restricted(self, g, src_groups, tgt_groups):  # interface_system.py:148-162
        src = set(src_groups)
        return self._run(g, [s for s in self.lat.subs if s[0] + s[1] in src], set(tgt_groups))
