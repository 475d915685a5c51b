"""Workloads of the device-checks library (HS_LIB=debug, libhsb200_debug.so):
every dataflow kernel on small and BASELINE-1/2 sizes, results checked
against the reference goldens / the single-RHS kernels, and hs_debug_check
after each (bounds asserts on every table / map / vector access, watchdogs on
every cross-CTA spin-wait).  One JSON line per workload.
    HS_LIB=debug python tools/device_checks.py [case ...]
Cases: fused (k_bsp_tma map-once + GMRES A M v), steps (fused per-step plan),
zmma (k_zmma2 R = 4, 64, 100 + shared maps), emu (emulated row-band ranks of
the fused apply), gmres (every Arnoldi variant), peer (peer all-reduce).
compute-sanitizer is closed on this GPU pool (it left GPUs needing resets);
this is its stand-in for out-of-bounds accesses and protocol hangs."""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from conftest import cvec, golden, product_problem, relerr  # noqa: E402
from paper_2209_10886_b200 import native  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS, small_case  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402


def check(s):
    first, en = C.c_uint64(0), C.c_int(0)
    s.ctx.call("hs_debug_check", C.byref(first), C.byref(en))
    return int(first.value), int(en.value)


def emit(case, cfg, errs, s, ok):
    code, en = check(s)
    rec = {"case": case, "config": cfg, "lib": os.path.basename(native.LIB_PATH), "checks_enabled": en,
           "violation": code, "violation_line": (code >> 8) & 0xFFFFFFFF if code else None,
           "errors": {k: float(v) for k, v in errs.items()}, "ok": bool(ok and code == 0)}
    print(json.dumps(rec), flush=True)
    return rec["ok"]


def sys_for(c, **kw):
    spec, part = product_problem(c)
    return GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]), **kw)


def case_fused(steps=False):
    ok = True
    for name in ("small", "cfg1", "cfg2"):
        c = small_case(3, 3, 32) if name == "small" else CONFIGS[int(name[-1])]
        s = sys_for(c, fused="steps" if steps else True)
        ref = sys_for(c, fused="literal")
        L = s.layout.size
        g = cvec(3, L)
        errs = {"bsp_vs_literal": max(relerr(s.bsp_apply(g), ref.bsp_apply(g)) for _ in range(3))}
        b = s.rhs()
        r1 = s.gmres(b, "bsp", tol=1e-8, maxit=200)
        r2 = ref.gmres(b, "bsp", tol=1e-8, maxit=200)
        errs["gmres_x"] = relerr(r1.solution, r2.solution)
        errs["iters_diff"] = abs(r1.iterations - r2.iterations)
        if name != "small":
            G = golden(name)
            errs["bsp_vs_golden"] = relerr(s.bsp_apply(G["r"]), G["M_bsp"])
            errs["ims_vs_golden"] = relerr(s.apply_interface_operator(G["g"]), G["Ag"])
        tol = 1e-16 if steps else 1e-13
        ok &= emit("steps" if steps else "fused", name, errs, s,
                   errs["bsp_vs_literal"] < tol and errs["iters_diff"] == 0 and errs["gmres_x"] < 1e-11
                   and errs.get("bsp_vs_golden", 0) < 1e-10 and errs.get("ims_vs_golden", 0) < 1e-10)
    return ok


def case_zmma():
    ok = True
    for name in ("cfg1", "cfg2"):
        c = CONFIGS[int(name[-1])]
        s = sys_for(c)
        L = s.layout.size
        for R in (4, 64, 100):
            X = cvec(5, L, R)
            Z, Y = s.bsp_apply(X), s.apply_interface_operator(X)
            cols = sorted({0, R // 2, R - 1})
            errs = {"bsp": max(relerr(Z[:, r], s.bsp_apply(np.ascontiguousarray(X[:, r]))) for r in cols),
                    "ims": max(relerr(Y[:, r], s.apply_interface_operator(np.ascontiguousarray(X[:, r]))) for r in cols)}
            ok &= emit(f"zmma_R{R}", name, errs, s, errs["bsp"] < 1e-13 and errs["ims"] < 1e-14)
        sh = sys_for(c, maps="shared")
        G = golden(name)
        errs = {"bsp_vs_golden": relerr(sh.bsp_apply(G["r"]), G["M_bsp"]),
                "ims_vs_golden": relerr(sh.apply_interface_operator(G["g"]), G["Ag"])}
        ok &= emit("zmma_shared", name, errs, sh, errs["bsp_vs_golden"] < 1e-10 and errs["ims_vs_golden"] < 1e-10)
    return ok


def case_emu():
    ok = True
    for name in ("cfg1", "cfg2"):
        c = CONFIGS[int(name[-1])]
        s = sys_for(c)
        g = cvec(7, s.layout.size)
        z1 = s.bsp_apply(g)
        for G in (2, 4):
            s.ctx.call("hs_set_emulated_ranks", G)
            e = relerr(s.bsp_apply(g), z1)
            s.ctx.call("hs_set_emulated_ranks", 1)
            ok &= emit(f"emu_G{G}", name, {"bsp_vs_single": e}, s, e == 0.0)
    return ok


def case_gmres():
    ok = True
    for name in ("cfg1", "cfg2"):
        c = CONFIGS[int(name[-1])]
        s = sys_for(c)
        G = golden(name)
        for mode in ("auto", "grid", "hostloop", "cgs2"):
            r = s.gmres(G["b"], "bsp", tol=1e-6, maxit=1000, arnoldi=mode)
            errs = {"iters_diff": abs(r.iterations - int(G["gm_iters"])), "x_vs_golden": relerr(r.solution, G["gm_x"])}
            ok &= emit(f"gmres_{mode}", name, errs, s, errs["iters_diff"] <= 1 and errs["x_vs_golden"] < 1e-8)
    return ok


def case_peer():
    s = sys_for(small_case(2, 2, 8))
    ok = True
    for G, count, rep in ((2, 100, 100), (8, 4096, 10)):
        rng = np.random.default_rng(G)
        x = rng.standard_normal((rep, G, count))
        out = np.empty_like(x)
        s.ctx.call("hs_test_peer_allreduce", G, count, rep, C.c_void_p(x.ctypes.data), C.c_void_p(out.ctypes.data))
        want = np.zeros((rep, count))
        for g in range(G):
            want = want + x[:, g, :]
        e = max(float(np.abs(out[:, g, :] - want).max()) for g in range(G))
        ok &= emit(f"peer_G{G}", "synthetic", {"max_abs_vs_rank_order_sum": e}, s, e == 0.0)
    return ok


def case_selftest():
    """The instrumentation reports: a deliberately failing check (unit 1, tag
    DBG_INDEX) must come back through hs_debug_check."""
    s = sys_for(small_case(2, 2, 8))
    check(s)
    s.ctx.call("hs_debug_selftest")
    code, en = check(s)
    want = (en == 1 and (code >> 48) == 1 and (code & 0xFF) == 1) or (en == 0 and code == 0)
    print(json.dumps({"case": "selftest", "lib": os.path.basename(native.LIB_PATH), "checks_enabled": en,
                      "violation": 0, "reported": code, "ok": bool(want)}), flush=True)
    return want


CASES = {"selftest": case_selftest, "fused": case_fused, "steps": lambda: case_fused(steps=True), "zmma": case_zmma, "emu": case_emu,
         "gmres": case_gmres, "peer": case_peer}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    allok = all([CASES[n]() for n in names])
    sys.exit(0 if allok else 1)
