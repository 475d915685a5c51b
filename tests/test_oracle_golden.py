"""CPU: the oracle restatement is pinned to golden vectors produced by the real
reference (tests/golden/make_golden.py).  The SuperLU back end must reproduce
the reference bit for bit (same matrix, same SciPy SuperLU); the dense
Schur-map back end (the accurate oracle the GPU mirrors) within the
reference's own scatterer-subdomain error."""

import numpy as np
import pytest

from conftest import golden, oracle_problem, relerr
from paper_2209_10886_b200.configs import CONFIGS, small_case

from oracle import Interface, Preconditioner, gmres
from oracle.fd import Subdomain, mono_solve
from oracle.lattice import FACE_NAMES, Lattice, reference_windows

SMALL = {
    "small_2x2": small_case(2, 2, 8),
    "small_3x3": small_case(3, 3, 8),
    "small_3x2": small_case(3, 2, 12),
    "small_1x4": small_case(1, 4, 8),
    "cfg1": CONFIGS[1],
}

_ITF = {}


def itf(name, backend="superlu"):
    key = (name, backend)
    if key not in _ITF:
        prob, lat = oracle_problem(SMALL[name] if name in SMALL else CONFIGS[2])
        _ITF[key] = Interface(prob, lat, backend=backend)
    return _ITF[key]


def test_lattice_tables_match_reference():
    G = golden("lattice")
    for key in G.files:
        if not key.startswith("pairs_"):
            continue
        n1, n2 = map(int, key[6:].split("x"))
        lat = Lattice(n1, n2)
        tab = np.array([[o[0], o[1], j[0], j[1]] for o, j in lat.pairs], dtype=np.int32).reshape(-1, 4)
        assert np.array_equal(tab, G[key]), key
        for kind in ("lower", "upper"):
            w = np.array(reference_windows(n1, lat.n_groups, kind), dtype=np.int32).reshape(-1, 2)
            assert np.array_equal(w, G[f"win_{kind}_{n1}x{n2}"]), (key, kind)


@pytest.mark.parametrize("name", list(SMALL))
def test_superlu_oracle_bitwise(name):
    G = golden(name)
    I = itf(name)
    assert np.array_equal(I.apply_S(G["g"]), G["Sg"])
    assert np.array_equal(I.apply_A(G["g"]), G["Ag"])
    assert np.array_equal(I.rhs(), G["b"])
    for key in G.files:
        if key.startswith("R_"):
            _, a, b = key.split("_")
            assert np.array_equal(I.restricted(G["g"], {int(a)}, {int(b)}), G[key]), key


@pytest.mark.parametrize("name", list(SMALL))
def test_local_solve_and_traces(name):
    G = golden(name)
    I = itf(name)
    for key in G.files:
        if not (key.startswith("local_") and key.endswith("_u")):
            continue
        _, a, b, _u = key.split("_")
        sub = (int(a), int(b))
        op = I.ops[sub]
        tr = {}
        for f in op.iface:
            tr[f] = G[f"local_{a}_{b}_in_{FACE_NAMES[f]}"]
        u = op.solve(tr)
        assert np.array_equal(u, G[key])
        for f in op.iface:
            assert np.array_equal(op.outgoing(u, tr[f], f), G[f"local_{a}_{b}_out_{FACE_NAMES[f]}"])
            # out = in - 2 (u_g - u_c)/h entry-wise
            uc = u[op.faces[f]]
            ug = (tr[f] + op.s * uc) / op.d
            alt = tr[f] - 2 * (ug - uc) / op.prob.h
            assert np.allclose(op.outgoing(u, tr[f], f), alt, rtol=1e-14, atol=1e-14 * np.abs(alt).max())


@pytest.mark.parametrize("name", ["small_2x2", "small_3x3", "small_3x2", "small_1x4"])
def test_dense_and_mono(name):
    G = golden(name)
    I = itf(name)
    assert np.array_equal(I.dense_S(), G["S_dense"])
    if "mono" in G.files:
        prob, lat = oracle_problem(SMALL[name])
        assert np.array_equal(mono_solve(prob, lat), G["mono"])


@pytest.mark.parametrize("name", list(SMALL))
def test_sweeps_match_spec_restatement_on_reference_S(name):
    G = golden(name)
    I = itf(name)
    r = G["r"]
    assert np.array_equal(Preconditioner(I, "sp")(r), G["M_sp"])
    pc = Preconditioner(I, "bsp")
    assert np.array_equal(pc(r), G["M_bsp"])
    assert np.array_equal(pc.bj_half_apply(r, "forward"), G["half_fwd"])
    assert np.array_equal(pc.bj_half_apply(r, "backward"), G["half_bwd"])
    assert np.array_equal(Preconditioner(I, "bsp", seam="literal")(r), G["M_bsp_literal"])
    assert np.array_equal(Preconditioner(I, "bsp", intermediate_residual=False)(r), G["M_bsp_nores"])
    assert np.array_equal(Preconditioner(I, "bsp", blocks=1)(r), G["M_bsp1"])


@pytest.mark.parametrize("name", list(SMALL))
def test_gmres_matches_golden(name):
    G = golden(name)
    I = itf(name)
    res = gmres(I.apply_A, Preconditioner(I, "bsp"), I.rhs(), tol=1e-6, maxit=1000)
    assert res.iterations == int(G["gm_iters"])
    assert np.array_equal(res.x, G["gm_x"])
    assert np.array_equal(np.array(res.history), G["gm_hist"])


@pytest.mark.parametrize("name", ["small_2x2", "small_3x3", "cfg1"])
def test_schur_oracle_close_to_reference(name):
    """The accurate (Dirichlet-eliminated) Schur-map oracle against the
    reference: generic subdomains to rounding, the scatterer subdomain within
    the reference's own SuperLU error."""
    G = golden(name)
    I = itf(name, "schur")
    assert relerr(I.apply_S(G["g"]), G["Sg"]) < 1e-11
    pc = Preconditioner(I, "bsp")
    assert relerr(pc(G["r"]), G["M_bsp"]) < 1e-11


def test_cfg2_apply_bitwise():
    G = golden("cfg2")
    prob, lat = oracle_problem(CONFIGS[2])
    I = Interface(prob, lat)
    assert np.array_equal(I.apply_A(G["g"]), G["Ag"])
    assert np.array_equal(I.rhs(), G["b"])


def test_subdomain_matrix_is_reference_matrix():
    """helmholtz_matrix restates _assemble_grid (discretization.py:221-256);
    spot-check structure: symmetric apart from Dirichlet rows."""
    prob, lat = oracle_problem(SMALL["small_2x2"])
    op = Subdomain(prob, lat, (1, 1))
    A = op.matrix.toarray()
    D = np.zeros(A.shape[0], bool)
    D[op.dcells] = True
    S = A - A.T
    assert np.abs(S[~D][:, ~D]).max() == 0.0


def test_shared_factor_parallel_oracle_bitwise_cfg2_sweep():
    """The CPU baseline's machinery (oracle.parallel over Interface(share_factors=
    True): 2 SuperLU factors, forked workers) reproduces the reference's cfg2
    block-sweep goldens bit for bit (make_golden.py --cfg2-sweep)."""
    from oracle.parallel import ParInterface
    G = golden("cfg2")
    if "M_bsp_p8" not in G.files:
        pytest.skip("cfg2 golden without the block sweep")
    prob, lat = oracle_problem(CONFIGS[2])
    I = Interface(prob, lat, share_factors=True)
    assert I.n_factors == 2
    with ParInterface(I, 2) as P:
        for p in (4, 8):
            assert np.array_equal(Preconditioner(P, "bsp", blocks=p)(G["r"]), G[f"M_bsp_p{p}"]), p
        assert np.array_equal(P.apply_A(G["g"]), G["Ag"])
        assert np.array_equal(P.restricted(G["g"], {5}, {6}), G["R_5_6"])


def test_cfg3_shared_factor_record():
    """Record of make_golden.py --check-cfg3: the shared-factor, process-parallel
    reference harness reproduced the cfg3 golden (one factor per subdomain,
    serial loop) bit for bit -- the premise of the cfg5 golden."""
    import json
    import os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "cfg3_shared_check.json")) as f:
        rep = json.load(f)
    for k in ("b", "Ag", "M_bsp4", "gm_x", "gm_hist"):
        assert rep[k]["bitwise_equal"] and rep[k]["max_abs_diff"] == 0.0, k
    assert rep["gm_iters"]["golden"] == rep["gm_iters"]["shared"] == 67


def test_cfg5_golden_reference_vs_accurate_oracle():
    """The cfg5 golden (reference arithmetic, shared SuperLU factors) and the
    accurate oracle's values on the same inputs agree within the reference's
    scatterer-subdomain floor: same iteration count, x within
    the north_star bar of 1e-8."""
    G = golden("cfg5")
    assert int(G["gm_iters"]) == int(G["acc_iters"]) == 107
    x = G["gm_x"]
    assert np.linalg.norm(G["acc_dx"]) / np.linalg.norm(x) < 5e-9
    assert np.linalg.norm(G["acc_dAg"]) / np.linalg.norm(G["Ag"]) < 1e-9
    assert np.linalg.norm(G["acc_dbsp"]) / np.linalg.norm(G["M_bsp8"]) < 2e-9
    assert G["gm_hist"][-1] <= 1e-6 * G["gm_hist"][0] < G["gm_hist"][-2]
