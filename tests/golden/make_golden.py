"""Generate golden fixtures from the REAL reference package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--cfg3]
    python tests/golden/make_golden.py --check-cfg3   # shared-factor harness == cfg3 golden, bitwise
    python tests/golden/make_golden.py --cfg2-sweep   # cfg2 block counts p = 1, 2, 4, 8
    python tests/golden/make_golden.py --cfg5         # headline config, ~32 min on 8 cores
    python tests/golden/make_golden.py --cfg5-acc     # add the accurate-oracle terms to cfg5.npz

Writes tests/golden/*.npz.  What is pinned:
  * lattice.npz   : m-order pair tables and reference windows for several lattices
                    (indexing.py:79-179);
  * small_*.npz   : seeded S g, (I-S) g, restricted applies, b, the dense S
                    (interface_system.py:98-175) for 2x2 / 3x3 / 3x2 at n=8 and
                    cfg1, plus single-subdomain solve_local/extract outputs
                    (discretization.py:264-312);
  * sweeps_*.npz  : SP / BSP applies and the full GMRES run, evaluated by the
                    SPEC restatement (oracle.sweeps / oracle.gmres) whose every S
                    application is the reference's InterfaceSystem.restricted_apply
                    / apply_interface_operator;
  * mono_*.npz    : mono_solve fields (discretization.py:335-370).
  * cfg5.npz / cfg2 sweep / cfg3 check: the same reference arithmetic run by
    `refpar` (shared bitwise-identical SuperLU factors + forked workers calling
    the reference's own `_scatter_one`); see tests/golden/refpar.py.
The reference package is never imported by the product, the GPU tests or bench.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")

from helmsweep import indexing as ref_idx  # noqa: E402
from helmsweep import discretization as ref_disc  # noqa: E402
from helmsweep import interface_system as ref_is  # noqa: E402

from oracle.gmres import gmres  # noqa: E402
from oracle.lattice import Lattice  # noqa: E402
from oracle.sweeps import Preconditioner  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS, small_case  # noqa: E402


class RefAdapter:
    """Presents the reference InterfaceSystem with the oracle Interface API so the
    SPEC restatement of the sweeps runs on the reference's own S applications."""

    def __init__(self, system, lat):
        self.sys = system
        self.lat = lat
        self.n = system.layout.n
        self.size = system.layout.size

    def restricted(self, g, src, tgt):
        g = np.asarray(g)
        if g.ndim == 1:
            return self.sys.restricted_apply(g, src, tgt)
        return np.stack([self.sys.restricted_apply(g[:, r], src, tgt) for r in range(g.shape[1])], 1)

    def apply_A(self, g):
        g = np.asarray(g)
        if g.ndim == 1:
            return self.sys.apply_interface_operator(g)
        return np.stack([self.sys.apply_interface_operator(g[:, r]) for r in range(g.shape[1])], 1)


def ref_system(c):
    spec = ref_disc.ProblemSpec(
        kappa=c["kappa"], cells_per_side=c["n"], subdomain_side=c["side"],
        scatterer=None if c["center"] is None else ref_disc.Scatterer(tuple(c["center"]), c["radius"]),
        incident_direction=(float(np.cos(c["angle"])), float(np.sin(c["angle"]))))
    part = ref_idx.Partition(c["n1"], c["n2"])
    return spec, part, ref_is.InterfaceSystem(spec, part)


def rng_vec(seed, size, R=None):
    rng = np.random.default_rng(seed)
    shape = (size,) if R is None else (size, R)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def lattice_fixture():
    out = {}
    for n1, n2 in [(1, 1), (2, 2), (3, 3), (4, 4), (5, 5), (5, 10), (1, 5), (6, 3), (8, 8), (16, 16), (32, 16)]:
        p = ref_idx.Partition(n1, n2)
        tab = np.array([[a.owner.i1, a.owner.i2, a.neighbor.i1, a.neighbor.i2] for a in p.pairs], dtype=np.int32).reshape(-1, 4)
        out[f"pairs_{n1}x{n2}"] = tab
        for kind in ("lower", "upper"):
            out[f"win_{kind}_{n1}x{n2}"] = np.array([[w.lo, w.hi] for w in ref_idx.build_windows(p, kind)], dtype=np.int32).reshape(-1, 2)
    np.savez_compressed(os.path.join(HERE, "lattice.npz"), **out)


def apply_fixture(name, c, dense=False, mono=False, gm=True, seeds=(1, 2)):
    t0 = time.time()
    spec, part, sysr = ref_system(c)
    lat = Lattice(c["n1"], c["n2"])
    L = sysr.layout.size
    out = {"L": L}
    lifts = sysr.compute_liftings()
    b = sysr.assemble_rhs(lifts)
    out["b"] = b
    g = rng_vec(seeds[0], L)
    out["g"] = g
    out["Sg"] = sysr.apply_scattering(g)
    out["Ag"] = sysr.apply_interface_operator(g)
    ng = part.n_groups
    gams = range(3, ng + 2) if L < 20000 else (3, ng // 2 + 1, ng + 1)
    for gam in gams:
        out[f"R_{gam - 1}_{gam}"] = sysr.restricted_apply(g, {gam - 1}, {gam})
        out[f"R_{gam}_{gam - 1}"] = sysr.restricted_apply(g, {gam}, {gam - 1})
    if dense:
        out["S_dense"] = sysr.materialize_dense()
    if mono:
        out["mono"] = ref_disc.mono_solve(spec, part)
    # single-subdomain local solve + outgoing traces (discretization.py:264-312)
    home = ref_disc.scatterer_subdomain(spec, part)
    for sub in {tuple(part.subdomains[0]), tuple(part.subdomains[-1])} | ({tuple(home)} if home else set()):
        op = sysr.operators[ref_idx.MultiIndex(*sub)]
        rng = np.random.default_rng(7)
        inc = {f: rng.standard_normal(c["n"]) + 1j * rng.standard_normal(c["n"]) for f in op.interface_faces}
        fld = ref_disc.solve_local(op, inc)
        out[f"local_{sub[0]}_{sub[1]}_u"] = fld.values
        for f in op.interface_faces:
            out[f"local_{sub[0]}_{sub[1]}_in_{f}"] = inc[f]
            out[f"local_{sub[0]}_{sub[1]}_out_{f}"] = ref_disc.extract_outgoing_trace(op, fld, inc[f], f)
    # sweeps on the reference S
    adap = RefAdapter(sysr, lat)
    r = rng_vec(seeds[1], L)
    out["r"] = r
    for kind, blocks in [("sp", None), ("bsp", None), ("bsp", 1)] + ([("bsp", c["blocks"])] if c.get("blocks") else []):
        pc = Preconditioner(adap, kind, blocks=blocks)
        tag = f"{kind}{'' if blocks is None else blocks}"
        out[f"M_{tag}"] = pc(r)
        if kind == "bsp" and blocks is None:
            out["M_bsp_literal"] = Preconditioner(adap, "bsp", seam="literal")(r)
            out["M_bsp_nores"] = Preconditioner(adap, "bsp", intermediate_residual=False)(r)
            out["half_fwd"] = pc.bj_half_apply(r, "forward")
            out["half_bwd"] = pc.bj_half_apply(r, "backward")
    if gm:
        pc = Preconditioner(adap, "bsp", blocks=c.get("blocks"))
        t1 = time.time()
        res = gmres(adap.apply_A, pc, b, tol=c.get("tol", 1e-6), maxit=1000)
        out["gm_x"] = res.x
        out["gm_iters"] = res.iterations
        out["gm_hist"] = np.array(res.history)
        out["gm_time"] = time.time() - t1
        print(f"{name}: gmres {res.iterations} it, {time.time() - t1:.1f}s")
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: L={L} done in {time.time() - t0:.1f}s")


def par_system(c, workers):
    """Reference system with shared factors, driven by forked workers (refpar)."""
    from refpar import ParAdapter, shared_splu
    t0 = time.time()
    with shared_splu(ref_disc) as st:
        spec, part, sysr = ref_system(c)
    print(f"{c['name']}: reference system built in {time.time() - t0:.1f}s "
          f"({st['factor']} SuperLU factorisations, {st['reuse']} reused)", flush=True)
    return spec, part, sysr, ParAdapter(sysr, Lattice(c["n1"], c["n2"]), workers)


def _gmres_record(adap, b, blocks, tol, out, suffix=""):
    pc = Preconditioner(adap, "bsp", blocks=blocks)
    t1 = time.time()
    res = gmres(adap.apply_A, pc, b, tol=tol, maxit=1000)
    out[f"gm_x{suffix}"] = res.x
    out[f"gm_iters{suffix}"] = res.iterations
    out[f"gm_hist{suffix}"] = np.array(res.history)
    out[f"gm_time{suffix}"] = time.time() - t1
    print(f"  gmres{suffix}: {res.iterations} it, converged {res.converged}, {time.time() - t1:.1f}s", flush=True)
    return res


def check_cfg3(workers):
    """The shared-factor, process-parallel harness reproduces the committed cfg3
    golden (one SuperLU factor per subdomain, serial reference loop) bit for bit."""
    import json
    G = np.load(os.path.join(HERE, "cfg3.npz"))
    c = CONFIGS[3]
    spec, part, sysr, adap = par_system(c, workers)
    L = sysr.layout.size
    out = {}
    out["b"] = sysr.assemble_rhs(sysr.compute_liftings())
    out["Ag"] = adap.apply_A(rng_vec(int(G["seed_g"]), L))
    out["M_bsp4"] = Preconditioner(adap, "bsp", blocks=4)(rng_vec(int(G["seed_r"]), L))
    _gmres_record(adap, out["b"], 4, 1e-6, out)
    adap.close()
    rep = {}
    for k in ("b", "Ag", "M_bsp4", "gm_x", "gm_hist"):
        a, g = np.asarray(out[k]), np.asarray(G[k])
        rep[k] = {"bitwise_equal": bool(a.shape == g.shape and np.array_equal(a, g)),
                  "max_abs_diff": float(np.abs(a - g).max()) if a.shape == g.shape else None}
    rep["gm_iters"] = {"golden": int(G["gm_iters"]), "shared": int(out["gm_iters"])}
    rep["workers"] = adap.workers
    rep["gmres_s"] = float(out["gm_time"])
    print(json.dumps(rep, indent=1))
    with open(os.path.join(HERE, "cfg3_shared_check.json"), "w") as f:
        json.dump(rep, f, indent=1)
        f.write("\n")
    assert all(v["bitwise_equal"] for k, v in rep.items() if isinstance(v, dict) and "bitwise_equal" in v)
    assert rep["gm_iters"]["golden"] == rep["gm_iters"]["shared"]


def cfg2_sweep(workers):
    """cfg2 block counts p = 1, 2, 4, 8 through the reference's restricted_apply
    (windows: SURVEY.md §8d rules (i)-(iii)); keys added to cfg2.npz."""
    G = dict(np.load(os.path.join(HERE, "cfg2.npz")))
    c = CONFIGS[2]
    spec, part, sysr, adap = par_system(c, workers)
    r = G["r"]
    b = G["b"]
    for p in (1, 2, 4, 8):
        z = Preconditioner(adap, "bsp", blocks=p)(r)
        G[f"M_bsp_p{p}"] = z
        out = {}
        _gmres_record(adap, b, p, 1e-6, out, suffix=f"_p{p}")
        G.update(out)
    adap.close()
    assert np.array_equal(G["M_bsp_p1"], G["M_bsp1"]) and np.array_equal(G["M_bsp_p2"], G["M_bsp"])
    np.savez_compressed(os.path.join(HERE, "cfg2.npz"), **G)


def cfg5_fixture(workers):
    """Headline config: b, seeded (I-S) g and BSP z, and the full GMRES run in
    the reference arithmetic; plus the accurate (Dirichlet-eliminated Schur map)
    oracle's solution, stored as its complex64 difference from the reference x."""
    from oracle import Interface
    c = CONFIGS[5]
    t0 = time.time()
    spec, part, sysr, adap = par_system(c, workers)
    L = sysr.layout.size
    out = {"L": L, "seed_g": 1, "seed_r": 2}
    out["b"] = sysr.assemble_rhs(sysr.compute_liftings())
    t1 = time.time()
    out["Ag"] = adap.apply_A(rng_vec(1, L))
    out["t_Ag"] = time.time() - t1
    t1 = time.time()
    out["M_bsp8"] = Preconditioner(adap, "bsp", blocks=8)(rng_vec(2, L))
    out["t_bsp"] = time.time() - t1
    print(f"cfg5: applies done ({out['t_Ag']:.1f}s, {out['t_bsp']:.1f}s)", flush=True)
    np.savez(os.path.join(HERE, "cfg5_partial.npz"), **out)
    _gmres_record(adap, out["b"], 8, 1e-6, out)
    adap.close()
    out["workers"] = adap.workers
    out.update(cfg5_accurate_terms(out))
    np.savez_compressed(os.path.join(HERE, "cfg5.npz"), **out)
    os.remove(os.path.join(HERE, "cfg5_partial.npz"))
    print(f"cfg5: done in {time.time() - t0:.1f}s; accurate oracle {int(out['acc_iters'])} it", flush=True)


def cfg5_accurate_terms(G):
    """The accurate (Dirichlet-eliminated Schur map) oracle on the golden's own
    inputs, stored as complex64 differences from the reference values (the
    differences are ~1e-10..1e-8 of the values, so complex64 keeps them to
    ~1e-17 absolute): b, (I-S) g, BSP z and the GMRES solution from the
    reference's b."""
    from oracle import Interface
    from oracle.schur import lifting_traces
    c = CONFIGS[5]
    prob, lat = oracle_from(c)
    itf = Interface(prob, lat, backend="schur")
    L = itf.size
    home, tr = lifting_traces(prob, lat)
    b = np.zeros(L, complex)
    for f, j in lat.faces[home]:
        m = lat.m_index(j, home)
        b[(m - 1) * prob.n:m * prob.n] = tr[f]
    out = {"acc_db": (b - G["b"]).astype(np.complex64),
           "acc_dAg": (itf.apply_A(rng_vec(int(G["seed_g"]), L)) - G["Ag"]).astype(np.complex64),
           "acc_dbsp": (Preconditioner(itf, "bsp", blocks=8)(rng_vec(int(G["seed_r"]), L)) - G["M_bsp8"]).astype(
               np.complex64)}
    acc = gmres(itf.apply_A, Preconditioner(itf, "bsp", blocks=8), G["b"], tol=1e-6, maxit=1000)
    out["acc_iters"] = acc.iterations
    out["acc_dx"] = (acc.x - G["gm_x"]).astype(np.complex64)
    out["acc_hist"] = np.array(acc.history)
    return out


def cfg5_add_accurate():
    """Add the accurate-oracle terms to an existing cfg5.npz (no reference rerun)."""
    G = dict(np.load(os.path.join(HERE, "cfg5.npz")))
    G.update(cfg5_accurate_terms(G))
    np.savez_compressed(os.path.join(HERE, "cfg5.npz"), **G)
    print("cfg5: accurate-oracle terms added", int(G["acc_iters"]), "it", flush=True)


def oracle_from(c):
    from oracle import Problem
    ang = c["angle"] if c["angle"] is not None else 0.0
    prob = Problem(kappa=c["kappa"], n=c["n"], side=c["side"],
                   center=None if c["center"] is None else tuple(c["center"]), radius=c["radius"],
                   direction=(float(np.cos(ang)), float(np.sin(ang))))
    return prob, Lattice(c["n1"], c["n2"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg3", action="store_true", help="also run config 3 (about 8 minutes)")
    ap.add_argument("--check-cfg3", action="store_true")
    ap.add_argument("--cfg2-sweep", action="store_true")
    ap.add_argument("--cfg5", action="store_true")
    ap.add_argument("--cfg5-acc", action="store_true", help="add the accurate-oracle terms to cfg5.npz")
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    if a.check_cfg3 or a.cfg2_sweep or a.cfg5 or a.cfg5_acc:
        sys.path.insert(0, HERE)
        if a.check_cfg3:
            check_cfg3(a.workers)
        if a.cfg2_sweep:
            cfg2_sweep(a.workers)
        if a.cfg5:
            cfg5_fixture(a.workers)
        if a.cfg5_acc:
            cfg5_add_accurate()
        return
    if a.only in (None, "lattice"):
        lattice_fixture()
    jobs = [
        ("small_2x2", small_case(2, 2, 8), dict(dense=True, mono=True)),
        ("small_3x3", small_case(3, 3, 8), dict(dense=True, mono=True)),
        ("small_3x2", small_case(3, 2, 12), dict(dense=True, mono=True)),
        ("small_1x4", small_case(1, 4, 8), dict(dense=True)),
        ("cfg1", CONFIGS[1], dict(mono=True)),
        ("cfg2", CONFIGS[2], dict()),
    ]
    if a.cfg3:
        jobs.append(("cfg3", CONFIGS[3], dict()))
    for name, c, kw in jobs:
        if a.only in (None, name):
            apply_fixture(name, c, **kw)


if __name__ == "__main__":
    main()
