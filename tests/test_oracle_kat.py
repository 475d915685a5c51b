"""CPU: SPEC.md known-answer tests and dense identities that pin the oracle's
restatement of the unshipped modules (preconditioner, krylov, driver)."""

import numpy as np
import pytest

from conftest import oracle_problem
from paper_2209_10886_b200.configs import small_case

from oracle import Interface, Preconditioner, gmres
from oracle.lattice import Lattice, reference_windows, windows
from oracle.pipeline import solve_problem
from oracle.sweeps import SchedulePlan, format_trace, step_schedule


# ---- indexing
def test_m_index_examples():
    lat = Lattice(2, 2)
    assert lat.m_index((1, 1), (1, 2)) == 1
    assert lat.m_index((1, 1), (2, 1)) == 2
    assert lat.m_index((1, 2), (1, 1)) == 3
    with pytest.raises(ValueError):
        lat.m_index((1, 1), (2, 2))


@pytest.mark.parametrize("n1,n2,ne,ng,pairs", [(2, 2, 4, 3, 8), (5, 10, 85, 14, 170), (1, 1, 0, 1, 0)])
def test_partition_counts(n1, n2, ne, ng, pairs):
    lat = Lattice(n1, n2)
    assert (lat.n_interfaces, lat.n_groups, lat.n_pairs) == (ne, ng, pairs)
    assert sum(len(v) for v in lat.groups.values()) == n1 * n2


def test_window_examples():
    assert reference_windows(5, 9, "lower") == [(2, 7), (7, 10)]
    assert reference_windows(5, 14, "lower") == [(2, 7), (7, 12), (12, 15)]
    assert reference_windows(5, 9, "upper") == [(5, 10), (2, 5)]


@pytest.mark.parametrize("n1,n2", [(4, 4), (8, 8), (16, 16), (32, 16), (5, 10), (1, 6), (6, 3)])
@pytest.mark.parametrize("p", [None, 1, 2, 3, 4, 7, 8])
def test_window_rule_invariants(n1, n2, p):
    ng = n1 + n2 - 1
    lw = windows(n1, n2, "lower", p)
    uw = windows(n1, n2, "upper", p)
    assert lw[0][0] == 2 and lw[-1][1] == ng + 1
    for a, b in zip(lw, lw[1:]):
        assert a[1] == b[0]  # one-group seams
    assert sorted((ng + 3 - hi, ng + 3 - lo) for lo, hi in lw) == sorted(uw)
    if p is not None:
        assert len(lw) == min(p, ng - 1)


def test_baseline_window_choices():
    """cfg2 p=4 and p=8, cfg3 p=4, cfg5 p=8."""
    assert windows(8, 8, "lower", 4) == [(2, 6), (6, 10), (10, 14), (14, 16)]
    assert windows(8, 8, "lower", 8) == [(2, 4), (4, 6), (6, 8), (8, 10), (10, 12), (12, 14), (14, 15), (15, 16)]
    assert windows(16, 16, "lower", 4) == [(2, 10), (10, 18), (18, 26), (26, 32)]
    assert windows(32, 16, "lower", 8)[:2] == [(2, 8), (8, 14)] and windows(32, 16, "lower", 8)[-1] == (44, 48)


# ---- step accounting
@pytest.mark.parametrize("n2,sp_ns", [(5, 16), (10, 26), (15, 36), (20, 46)])
def test_table1_step_counts(n2, sp_ns):
    lat = Lattice(5, n2)
    assert len(step_schedule(SchedulePlan(lat, "sp"))) == sp_ns
    assert len(step_schedule(SchedulePlan(lat, "bsp"))) == 10
    assert len(step_schedule(SchedulePlan(lat, "bsp", count_residual_steps=True))) == 11


def test_wavefronts_5x5():
    lat = Lattice(5, 5)
    sp = step_schedule(SchedulePlan(lat, "sp"))
    fw = [r for r in sp if r[1] == "forward"]
    assert len(fw) == 8
    for t, _, subs in fw:
        assert {a + b for a, b in subs} == {t + 1}
    bsp = step_schedule(SchedulePlan(lat, "bsp"))
    fw = [r for r in bsp if r[1] == "forward"]
    assert len(fw) == 5
    for t, _, subs in fw:
        want = {t + 1} | ({t + 6} if t <= 3 else set())
        assert {a + b for a, b in subs} == want
    assert format_trace(fw[:1]) == "step=1 phase=forward solves=(1,1);(2,5);(3,4);(4,3);(5,2)\n"
    assert format_trace(sp[:1]) == "step=1 phase=forward solves=(1,1)\n"
    assert step_schedule(SchedulePlan(Lattice(1, 1), "sp")) == []


# ---- dense identities (acceptance 2-3)
@pytest.fixture(scope="module")
def dense33():
    prob, lat = oracle_problem(small_case(3, 3, 8))
    itf = Interface(prob, lat)
    S = itf.dense_S()
    grp = np.repeat(np.asarray(lat.block_group()), itf.n)
    return itf, S, grp


def _blocks(S, grp, a, b):
    M = np.zeros_like(S)
    ia, ib = grp == a, grp == b
    M[np.ix_(ia, ib)] = S[np.ix_(ia, ib)]
    return M


def test_prop1_factorisation(dense33):
    itf, S, grp = dense33
    ng = itf.lat.n_groups
    N = S.shape[0]
    I = np.eye(N)
    SL = I - sum(_blocks(S, grp, g, g - 1) for g in range(3, ng + 2))
    SU = I - sum(_blocks(S, grp, g - 1, g) for g in range(3, ng + 2))
    P = I.copy()
    for g in range(3, ng + 2):
        P = P @ (I - _blocks(S, grp, g, g - 1))
    assert np.abs(P - SL).max() <= 1e-13 * max(1.0, np.abs(SL).max())
    Q = I.copy()
    for g in range(ng + 1, 2, -1):
        Q = Q @ (I - _blocks(S, grp, g - 1, g))
    assert np.abs(Q - SU).max() <= 1e-13 * max(1.0, np.abs(SU).max())
    # I - S = S_L + S_U - I; zero group-diagonal
    assert np.abs((I - S) - (SL + SU - I)).max() < 1e-13
    for g in range(2, ng + 2):
        assert np.abs(_blocks(S, grp, g, g)).max() == 0.0


def test_sweeps_vs_dense(dense33):
    itf, S, grp = dense33
    ng = itf.lat.n_groups
    N = S.shape[0]
    I = np.eye(N)
    SL = I - sum(_blocks(S, grp, g, g - 1) for g in range(3, ng + 2))
    SU = I - sum(_blocks(S, grp, g - 1, g) for g in range(3, ng + 2))
    rng = np.random.default_rng(0)
    r = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    pc = Preconditioner(itf, "sp")
    f = pc.forward_sweep(r)
    assert np.linalg.norm(f - np.linalg.solve(SL, r)) <= 1e-12 * np.linalg.norm(f)
    bk = pc.backward_sweep(r)
    assert np.linalg.norm(bk - np.linalg.solve(SU, r)) <= 1e-12 * np.linalg.norm(bk)
    z = pc.sgs_apply(r)
    assert np.linalg.norm(z - np.linalg.solve(SL @ SU, r)) <= 1e-11 * np.linalg.norm(z)
    # forward_sweep(S_L r) = r
    assert np.linalg.norm(pc.forward_sweep(SL @ r) - r) <= 1e-11 * np.linalg.norm(r)


@pytest.mark.parametrize("seam", ["dedup", "literal"])
def test_bsp_vs_dense_formula(dense33, seam):
    itf, S, grp = dense33
    N = S.shape[0]
    I = np.eye(N)
    ng = itf.lat.n_groups
    pc = Preconditioner(itf, "bsp", seam=seam)
    rng = np.random.default_rng(1)
    b = rng.standard_normal(N) + 1j * rng.standard_normal(N)

    def half(r, wins, lower):
        out = r.copy() if seam == "dedup" else np.zeros(N, complex)
        for lo, hi in wins:
            sel = np.flatnonzero((grp >= lo) & (grp <= hi))
            W = I[:, sel]
            if lower:
                Bm = I - sum(_blocks(S, grp, g, g - 1) for g in range(lo + 1, hi + 1))
            else:
                Bm = I - sum(_blocks(S, grp, g - 1, g) for g in range(lo + 1, hi + 1))
            B = W.T @ Bm @ W
            x = np.linalg.solve(B, W.T @ r)
            out += W @ (x - (W.T @ r if seam == "dedup" else 0))
        return out

    zl = half(b, pc.lower, True)
    rp = b - (I - S) @ zl
    z = zl + half(rp, pc.upper, False)
    got = pc(b)
    assert np.linalg.norm(got - z) <= 1e-11 * np.linalg.norm(z)
    assert ng >= 2


def test_bsp_one_window_equals_sp_per_half(dense33):
    itf, S, grp = dense33
    rng = np.random.default_rng(2)
    r = rng.standard_normal(S.shape[0]) + 1j * rng.standard_normal(S.shape[0])
    pc1 = Preconditioner(itf, "bsp", blocks=1)
    sp = Preconditioner(itf, "sp")
    assert np.linalg.norm(pc1.bj_half_apply(r, "forward") - sp.forward_sweep(r)) <= 1e-14 * np.linalg.norm(r)


def test_seam_modes_differ_only_on_seams(dense33):
    itf, S, grp = dense33
    rng = np.random.default_rng(3)
    r = rng.standard_normal(S.shape[0]) + 1j * rng.standard_normal(S.shape[0])
    d = Preconditioner(itf, "bsp", seam="dedup")
    l = Preconditioner(itf, "bsp", seam="literal")
    diff = l.bj_half_apply(r, "forward") - d.bj_half_apply(r, "forward")
    seams = {hi for lo, hi in d.lower[:-1]}
    mask = np.isin(grp, list(seams))
    assert np.allclose(diff[mask], r[mask], rtol=0, atol=1e-14)
    assert np.abs(diff[~mask]).max(initial=0.0) == 0.0


def test_preconditioners_are_linear(dense33):
    itf, S, grp = dense33
    rng = np.random.default_rng(4)
    N = S.shape[0]
    g1, g2 = [rng.standard_normal(N) + 1j * rng.standard_normal(N) for _ in range(2)]
    a, b = 0.7 - 0.2j, -1.3 + 0.5j
    for kind in ("sp", "bsp"):
        M = Preconditioner(itf, kind)
        lhs = M(a * g1 + b * g2)
        assert np.linalg.norm(lhs - (a * M(g1) + b * M(g2))) <= 1e-12 * np.linalg.norm(lhs)


# ---- GMRES (acceptance 5)
def test_gmres_identity_and_zero():
    b = np.arange(1, 7) + 1j
    res = gmres(lambda v: v, None, b, tol=1e-6)
    assert res.iterations == 1 and res.converged and np.allclose(res.x, b)
    res = gmres(lambda v: v, None, np.zeros(5, complex))
    assert res.iterations == 0 and res.converged and not np.any(res.x)


def test_gmres_dense_50():
    rng = np.random.default_rng(5)
    A = np.eye(50) * 8 + rng.standard_normal((50, 50)) + 1j * rng.standard_normal((50, 50))
    x0 = rng.standard_normal(50) + 1j * rng.standard_normal(50)
    b = A @ x0
    res = gmres(lambda v: A @ v, None, b, tol=1e-10, maxit=200)
    assert res.converged
    assert np.linalg.norm(res.x - x0) <= 1e-8 * np.linalg.norm(x0)
    hist = np.array(res.history)
    assert np.all(np.diff(hist) <= 1e-15)


def test_gmres_matrix_free_vs_dense():
    prob, lat = oracle_problem(small_case(2, 2, 8))
    itf = Interface(prob, lat)
    S = itf.dense_S()
    A = np.eye(S.shape[0]) - S
    pc = Preconditioner(itf, "sp")
    M = np.stack([pc(e) for e in np.eye(S.shape[0], dtype=complex)], axis=1)
    b = itf.rhs()
    r1 = gmres(itf.apply_A, pc, b, tol=1e-10, maxit=200)
    r2 = gmres(lambda v: A @ v, lambda v: M @ v, b, tol=1e-10, maxit=200)
    assert r1.iterations == r2.iterations
    np.testing.assert_allclose(r1.history, r2.history, rtol=1e-10, atol=1e-14)


# ---- driver (acceptance 4, 6, 9)
@pytest.mark.parametrize("n1,n2", [(2, 2), (3, 2)])
def test_mono_equivalence(n1, n2):
    prob, lat = oracle_problem(small_case(n1, n2, 20))
    rep = solve_problem(prob, lat, kind="sp", tol=1e-10, mono_check=True)
    assert rep.converged
    assert rep.error_vs_mono["max_rel"] <= 1e-8


def test_degenerate_cases():
    prob, lat = oracle_problem(small_case(1, 1, 8))
    rep = solve_problem(prob, lat, kind="sp", tol=1e-10, mono_check=True)
    assert rep.iterations == 0 and rep.error_vs_mono["max_rel"] <= 1e-13
    c = dict(small_case(2, 2, 8))
    c["center"] = None
    prob, lat = oracle_problem(c)
    rep = solve_problem(prob, lat, kind="bsp")
    assert rep.iterations == 0 and not np.any(rep.b) and not np.any(rep.x)


def test_convergence_trend():
    """Acceptance 6: kappa = 2 pi, n = 25, N1 = 5, N2 in {5, 10}."""
    out = {}
    for n2 in (5, 10):
        prob, lat = oracle_problem(small_case(5, n2, 25))
        for kind in ("sp", "bsp"):
            rep = solve_problem(prob, lat, kind=kind, tol=1e-6, maxit=500)
            assert rep.converged
            out[(n2, kind)] = (rep.iterations, rep.steps_per_iteration)
    for n2 in (5, 10):
        assert out[(n2, "bsp")][0] >= out[(n2, "sp")][0]
    sp, bsp = out[(10, "sp")], out[(10, "bsp")]
    assert bsp[0] * bsp[1] <= sp[0] * sp[1]
