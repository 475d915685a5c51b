"""Modelled strong scaling of the peer-memory fused apply (a MODEL, not a
measurement: this run has one GPU).

Every rank's tile list comes from the library (hs_fused_plan on a plan-only
context with nranks = G, the global ticket order filtered to the rank).  The
model replays the dataflow: each rank has `ctas` persistent CTAs that claim its
tickets in order; a tile starts when its CTA is free and every dependency
(block, count) has its count-th completion signal visible; it then takes
  fixed + streamed_bytes / per-CTA stream rate
and signals the blocks it completes.  A signal crossing GPUs (writer or reader
not on the block's owner) costs `lat` extra.  Each rank's makespan is also
bounded below by its bytes / HBM bandwidth.  The constants are calibrated on
the one-GPU traces (profiles/r01/fused_trace_cfg*.json): stream rate from
stream_us, fixed cost from wait + epilogue.

  python tools/scaling_model.py CFG [G ...] [--gmres ITERS]

--gmres ITERS adds the modelled GMRES time-to-solution: ITERS x the replayed
A M v plan (hs_fused_plan ims = 1) + the one-reduction CGS2 Arnoldi per
iteration k: two passes over the rank's V slice (2 (k+1) L/G x 16 B at the
HBM rate) + its fixed cost (calibrated on the one-GPU launch list,
profiles/r02/gmres_launches_cfg5.csv: 23 ms of Arnoldi for 107 iterations =
14 ms of streaming + ~80 us per iteration of launches / coefficients) + one
peer-memory all-reduce across ranks (~8 us: two NVLink latencies + a kernel).
"""
import bisect
import ctypes as C
import heapq
import json
import sys

import numpy as np

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from paper_2209_10886_b200 import native  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS  # noqa: E402
from paper_2209_10886_b200.indexing import window_ranges  # noqa: E402


def parse(v):
    out, i = [], 0
    while i < len(v):
        rec = [int(x) for x in v[i:i + 12]]
        nd = rec[11]
        deps = [(int(v[i + 12 + 2 * d]), int(v[i + 13 + 2 * d])) for d in range(nd)]
        out.append((rec, deps))
        i += 12 + 2 * nd
    return out


def plans(cfg, G, ims=0):
    c = CONFIGS[cfg]
    n = c["n"]
    out = []
    for g in range(G):
        ctx = native.Context(-1, c["n1"], c["n2"], n, 0.1, 1.0, 1j, rank=g, nranks=G)
        for k, kd in ((0, "lower"), (1, "upper")):
            w = window_ranges(c["n1"], c["n2"], kd, c["blocks"])
            lo, hi = native.i32([a for a, _ in w]), native.i32([b for _, b in w])
            ctx.call("hs_set_windows", k, native.iptr(lo), native.iptr(hi), len(w))
        cnt = C.c_int(0)
        ctx.call("hs_fused_plan", ims, g, None, 0, C.byref(cnt))
        buf = (C.c_int32 * cnt.value)()
        ctx.call("hs_fused_plan", ims, g, buf, cnt.value, C.byref(cnt))
        owner = ctx.block_owner()
        out.append(parse(np.frombuffer(buf, dtype=np.int32)))
    return out, owner, c


def lattice_maps(c):
    from oracle.lattice import Lattice
    return Lattice(c["n1"], c["n2"])


def tile_key(rec):
    return tuple(rec[:10])


def critical_tiles(cfg, frac, rate=31.6e9, fixed=3.0e-6):
    """Tiles whose longest path to the end of the apply is >= frac of the
    longest (the global plan, unlimited CTAs)."""
    pl, owner, c = plans(cfg, 1)
    lat_ = lattice_maps(c)
    n = c["n"]
    tl = pl[0]
    writers = {}
    dur = []
    for i, (rec, deps) in enumerate(tl):
        i1, i2, rlo, rhi, c0, c1, alt, row0, phase, flags, rmask, _ = rec
        rows = min(rhi, row0 + 32) - max(rlo, row0)
        dur.append(fixed + 16.0 * rows * (c1 - c0) / rate)
    succ = [[] for _ in tl]
    for i, (rec, deps) in enumerate(tl):
        for b, cnt in deps:
            for w in writers.get(b, [])[:cnt]:
                succ[w].append(i)
        i1, i2, rlo, rhi, c0, c1, alt, row0, phase, flags, rmask, _ = rec
        s = (i1, i2)
        if phase not in (3, 5):
            nlow = sum(1 for f, _ in lat_.faces[s] if f in (0, 1))
            r0, r1 = max(rlo, row0), min(rhi, row0 + 32)
            for f in range(r0 // n, (r1 - 1) // n + 1):
                if phase <= 1 or f < nlow:
                    writers.setdefault(lat_.m_index(lat_.faces[s][f][1], s) - 1, []).append(i)
    bl = [0.0] * len(tl)
    for i in range(len(tl) - 1, -1, -1):
        bl[i] = dur[i] + max((bl[j] for j in succ[i]), default=0.0)
    top = max(bl)
    return {tile_key(tl[i][0]) for i in range(len(tl)) if bl[i] >= frac * top}


def simulate(cfg, G, ctas=296, rate=31.6e9, fixed=3.0e-6, lat=3.0e-6, hbm=6.9e12, rate_max=None, split=False,
             split_set=None, ims=0):
    """rate: per-CTA stream rate under full load (calibrated); rate_max: the
    ring-latency limit of one CTA (5 x 16 KB in flight) when fewer CTAs share
    the HBM -- the rate of a tile is then min(rate_max, hbm / CTAs streaming at
    its start)."""
    pl, owner, c = plans(cfg, G, ims)
    lat_ = lattice_maps(c)
    n = c["n"]
    # global ticket order = merge of the rank lists by their global position: the
    # library keeps each rank's tiles in the one global order, so a k-way merge by
    # dependency-readiness is not needed -- replay round-robin by earliest claim
    signals = {}  # block -> sorted visible-at-owner times
    free = [[0.0] * ctas for _ in range(G)]
    for f in free:
        heapq.heapify(f)
    idx = [0] * G
    active = [[] for _ in range(G)]  # end times of the tiles streaming on each rank
    bytes_rank = [0.0] * G
    end_rank = [0.0] * G
    pending = sum(len(p) for p in pl)

    def sig_blocks(rec):
        i1, i2, rlo, rhi, c0, c1, alt, row0, phase, flags, rmask, _ = rec
        s = (i1, i2)
        if phase in (3, 5):
            return []
        nlow = sum(1 for f, _ in lat_.faces[s] if f in (0, 1))
        r0, r1 = max(rlo, row0), min(rhi, row0 + 32)
        return [lat_.m_index(lat_.faces[s][f][1], s) - 1 for f in range(r0 // n, (r1 - 1) // n + 1)
                if phase <= 1 or f < nlow]

    def dep_time(g, deps):
        t = 0.0
        for b, cnt in deps:
            lst = signals.get(b, [])
            if len(lst) < cnt:
                return None  # not all writers replayed yet
            t = max(t, lst[cnt - 1] + (lat if owner[b] != g else 0.0))
        return t

    while pending:
        progressed = False
        for g in range(G):
            while idx[g] < len(pl[g]):
                rec, deps = pl[g][idx[g]]
                dt = dep_time(g, deps)
                if dt is None:
                    break
                claim = heapq.heappop(free[g])
                i1, i2, rlo, rhi, c0, c1, alt, row0, phase, flags, rmask, _ = rec
                rows = min(rhi, row0 + 32) - max(rlo, row0)
                nb = 16.0 * rows * (c1 - c0)
                start = max(claim, dt)
                r = rate
                if rate_max:
                    act = active[g]
                    while act and act[0] <= start:
                        heapq.heappop(act)
                    r = min(rate_max, hbm / (len(act) + 1))
                if (split or (split_set is not None and tile_key(rec) in split_set)) and c1 - c0 >= 256:
                    # split-K: a second CTA streams the other column half; the
                    # later one adds the halves (fixed order) and finishes the rows
                    claim2 = heapq.heappop(free[g])
                    start2 = max(claim2, dt)
                    e1 = start + fixed + nb / 2 / r
                    e2 = start2 + fixed + nb / 2 / r
                    end = max(e1, e2) + 0.7e-6
                    heapq.heappush(free[g], min(e1, e2))
                    heapq.heappush(free[g], end)
                else:
                    end = start + fixed + nb / r
                    heapq.heappush(free[g], end)
                if rate_max:
                    heapq.heappush(active[g], end)
                bytes_rank[g] += nb
                end_rank[g] = max(end_rank[g], end)
                for b in sig_blocks(rec):
                    bisect.insort(signals.setdefault(b, []), end + (lat if owner[b] != g else 0.0))
                idx[g] += 1
                pending -= 1
                progressed = True
        if not progressed:
            raise RuntimeError("replay stuck: a dependency never completes")
    t = [max(e, b / hbm) for e, b in zip(end_rank, bytes_rank)]
    return max(t), t, bytes_rank


def main():
    cfg = int(sys.argv[1])
    Gs = [int(x) for x in sys.argv[2:] if not x.startswith("--")] or [1, 2, 4, 8]
    c = CONFIGS[cfg]
    calib = {5: dict(rate=31.6e9, fixed=3.0e-6), 3: dict(rate=38e9, fixed=3.5e-6)}.get(cfg, {})
    if "--shared-bw" in sys.argv:
        calib = dict(calib, rate_max=75e9)
    if "--split" in sys.argv:
        calib = dict(calib, split=True)
    for a in sys.argv:
        if a.startswith("--split-critical="):
            calib = dict(calib, split_set=critical_tiles(cfg, float(a.split("=")[1])))
    iters = None
    if "--gmres" in sys.argv:
        iters = int(sys.argv[sys.argv.index("--gmres") + 1])
        Gs = [G for G in Gs if G != iters]
    rows = []
    t1 = None
    g1 = None
    from oracle.lattice import Lattice
    L = Lattice(c["n1"], c["n2"]).n_pairs * c["n"]
    for G in Gs:
        if G > c["n2"]:
            continue
        T, per, by = simulate(cfg, G, **calib)
        t1 = T if G == 1 else t1
        row = {"G": G, "apply_ms": round(T * 1e3, 4), "per_rank_ms": [round(x * 1e3, 4) for x in per],
               "efficiency": round(t1 / (G * T), 3) if t1 else None}
        if iters:
            Tamv, _, _ = simulate(cfg, G, ims=1, **calib)
            hbm = 6.5e12
            arn = sum(2.0 * (k + 1) * (L / G) * 16.0 / hbm + 80e-6 + (8e-6 if G > 1 else 0.0) for k in range(iters))
            gm = iters * Tamv + arn
            g1 = gm if G == 1 else g1
            row.update({"amv_ms": round(Tamv * 1e3, 4), "arnoldi_ms": round(arn * 1e3, 2),
                        "gmres_ms": round(gm * 1e3, 2), "gmres_efficiency": round(g1 / (G * gm), 3) if g1 else None})
        rows.append(row)
    print(json.dumps({"config": cfg, "model": "tools/scaling_model.py (calibrated on the 1-GPU traces)",
                      "rows": rows}))


if __name__ == "__main__":
    main()
