"""GPU parity at the BASELINE sizes (configs 3, 4, 5).

cfg3: against the reference's own golden run (tests/golden/cfg3.npz: 67
iterations, x, (I-S) g, BSP apply); cfg5 likewise (tests/golden/cfg5.npz, 107
iterations) plus the accurate oracle's values on the same inputs.  cfg4: the 64-RHS batched GMRES against
per-angle oracle runs and, for angle k = 8 (= pi/4, config 2's angle), the
reference's cfg2 golden.  cfg5 (no full CPU run is feasible: ~2.2 h and 52 GB
in the reference as written; the golden comes from the shared-factor
harness): also the size-independent checks -- output blocks of sampled
subdomains against the reference arithmetic (SuperLU local solve + outgoing
traces, oracle/fd.py) and against the accurate Dirichlet-eliminated solve for
the scatterer subdomain, linearity, unitarity of the maps, the BSP identity
z = z_L + half_bwd(b - (I-S) z_L), and GMRES convergence with its true
residual.
"""

import math

import numpy as np
import pytest

from conftest import cvec, golden, oracle_problem, product_problem, relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200.configs import CONFIGS, angles  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

_S = {}


def system(k):
    if k not in _S:
        for key in list(_S):  # keep at most one big system resident
            del _S[key]
        spec, part = product_problem(CONFIGS[k])
        _S[k] = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=CONFIGS[k]["blocks"]))
    return _S[k]


def test_cfg3_vs_reference_golden():
    G = golden("cfg3")
    s = system(3)
    L = s.layout.size
    g = cvec(int(G["seed_g"]), L)
    r = cvec(int(G["seed_r"]), L)
    assert relerr(s.apply_interface_operator(g), G["Ag"]) < 1e-10
    # b: the reference's SuperLU lifting solve has componentwise backward error
    # 8e-9 at cfg3 (identity Dirichlet rows); the accurate
    # (eliminated) oracle has 3e-15 -> tight against the oracle, floor vs reference.
    from oracle.schur import lifting_traces
    prob, lat = oracle_problem(CONFIGS[3])
    home, tr = lifting_traces(prob, lat)
    b_acc = np.zeros(L, complex)
    for f, j in lat.faces[home]:
        m = lat.m_index(j, home)
        b_acc[(m - 1) * prob.n:m * prob.n] = tr[f]
    b = s.rhs()
    assert relerr(b, b_acc) < 1e-11
    assert relerr(b, G["b"]) < 5e-9
    z = s.bsp_apply(r)
    assert relerr(z, G["M_bsp4"]) < 1e-9  # reference floor (scatterer subdomain), amplified by the sweeps
    from oracle import Interface, Preconditioner
    itf = Interface(prob, lat, backend="schur")
    assert relerr(z, Preconditioner(itf, "bsp", blocks=4)(r)) < 1e-12
    res = s.gmres(G["b"], "bsp", tol=1e-6, maxit=1000)
    assert abs(res.iterations - int(G["gm_iters"])) <= 1, res.iterations
    assert relerr(res.solution, G["gm_x"]) < 1e-8
    assert relerr(s.apply_interface_operator(res.solution), G["b"]) < 1e-6


def test_cfg3_local_maps_vs_reference_local_solves():
    """T_s @ incoming = the reference's solve_local + extract_outgoing_trace."""
    G = golden("cfg3")
    s = system(3)
    faces = ("west", "south", "north", "east")
    for key in G.files:
        if not (key.startswith("local_") and key.endswith("_u")):
            continue
        _, a, b, _u = key.split("_")
        T = s.schur_map((int(a), int(b)))
        fs = [f for f in faces if f"local_{a}_{b}_in_{f}" in G.files]
        x = np.concatenate([G[f"local_{a}_{b}_in_{f}"] for f in fs])
        want = np.concatenate([G[f"local_{a}_{b}_out_{f}"] for f in fs])
        tol = 5e-9 if (int(a), int(b)) == (8, 8) else 1e-12  # reference SuperLU floor on the scatterer
        assert relerr(T @ x, want) < tol, (a, b, relerr(T @ x, want))


def test_cfg5_sampled_subdomains_vs_reference_arithmetic():
    from oracle.fd import Subdomain
    from oracle.schur import boundary_response
    s = system(5)
    prob, lat = oracle_problem(CONFIGS[5])
    L = s.layout.size
    g = cvec(21, L)
    Sg = s.apply_scattering(g)
    n = prob.n
    home = prob.home(lat)
    for sub in [(1, 1), (32, 16), (7, 9), (31, 2), home]:
        faces = lat.faces[sub]
        x = g[(lat.first_block[sub] - 1) * n:(lat.first_block[sub] - 1 + len(faces)) * n]
        tr = {f: x[q * n:(q + 1) * n] for q, (f, _) in enumerate(faces)}
        got = np.concatenate([Sg[(lat.m_index(j, sub) - 1) * n:lat.m_index(j, sub) * n] for f, j in faces])
        if sub == home:
            op = Subdomain(prob, lat, sub, factor=False)
            rhs = np.zeros(n * n, complex)
            for f, t in tr.items():
                rhs[op.faces[f]] += op.rhs_coeff * t
            u = boundary_response(prob, op.dcells, rhs[:, None])[:, 0]
            tol = 1e-11
        else:
            op = Subdomain(prob, lat, sub)
            u = op.solve(tr)
            tol = 1e-12
        want = np.concatenate([op.outgoing(u, tr[f], f) for f, _ in faces])
        assert relerr(got, want) < tol, (sub, relerr(got, want))


def test_cfg5_properties():
    s = system(5)
    L = s.layout.size
    g1, g2 = cvec(1, L), cvec(2, L)
    a, b = 0.3 - 1.1j, 2.0 + 0.5j
    lhs = s.apply_interface_operator(a * g1 + b * g2)
    rhs = a * s.apply_interface_operator(g1) + b * s.apply_interface_operator(g2)
    assert relerr(lhs, rhs) < 1e-13
    # the full 4-face map is unitary (lossless interior, tau = i kappa); boundary
    # subdomains' compact maps are sub-blocks (their exterior faces absorb)
    for sub in [(16, 8), (20, 10), (2, 2)]:
        T = s.schur_map(sub)
        assert T.shape[0] == 4 * 256
        assert np.abs(T.conj().T @ T - np.eye(T.shape[0])).max() < 1e-10
    T = s.schur_map((1, 1))
    assert np.linalg.norm(T, 2) <= 1 + 1e-10
    zl = s.bj_half_apply(g1, "forward")
    rp = g1 - s.apply_interface_operator(zl)
    z = zl + s.bj_half_apply(rp, "backward")
    assert relerr(s.bsp_apply(g1), z) < 1e-12


def test_cfg5_vs_reference_golden():
    """cfg5, the headline config, end to end against the reference arithmetic
    (tests/golden/cfg5.npz: the reference's own _scatter_one over shared,
    bitwise-identical SuperLU factors -- the harness reproduces the cfg3 golden
    bit for bit, cfg3_shared_check.json -- 107 GMRES iterations) and against
    the accurate (Dirichlet-eliminated Schur map) oracle on the same inputs.
    The reference floors come from its SuperLU solve on the scatterer
    subdomain: (I-S) g 2.1e-10, BSP z 4.5e-10, b 8.2e-9,
    x 1.9e-9 (accurate oracle vs reference)."""
    G = golden("cfg5")
    s = system(5)
    L = s.layout.size
    assert L == int(G["L"])
    g, r = cvec(int(G["seed_g"]), L), cvec(int(G["seed_r"]), L)
    Ag = s.apply_interface_operator(g)
    assert relerr(Ag, G["Ag"]) < 1e-9
    assert relerr(Ag, G["Ag"] + G["acc_dAg"]) < 1e-12
    z = s.bsp_apply(r)
    assert relerr(z, G["M_bsp8"]) < 2e-9
    assert relerr(z, G["M_bsp8"] + G["acc_dbsp"]) < 1e-12
    b = s.rhs()
    assert relerr(b, G["b"] + G["acc_db"]) < 1e-11
    assert relerr(b, G["b"]) < 5e-8
    res = s.gmres(G["b"], "bsp", tol=1e-6, maxit=1000)
    assert res.converged
    assert abs(res.iterations - int(G["gm_iters"])) <= 1, res.iterations
    assert relerr(res.solution, G["gm_x"]) < 1e-8
    assert relerr(res.solution, G["gm_x"] + G["acc_dx"]) < 1e-11
    k = min(res.iterations, int(G["acc_iters"]))
    np.testing.assert_allclose(res.history[:k + 1], G["acc_hist"][:k + 1], rtol=1e-10)
    np.testing.assert_allclose(res.history[:k + 1], G["gm_hist"][:k + 1], rtol=1e-8)
    assert relerr(s.apply_interface_operator(res.solution), G["b"]) < 1e-6
    assert np.all(np.diff(np.array(res.history)) <= 1e-12)


def test_cfg4_batched_gmres():
    from oracle import Interface, Preconditioner, gmres
    from oracle.schur import lifting_traces
    c = CONFIGS[4]
    s = system(4)
    dirs = [(math.cos(t), math.sin(t)) for t in angles(c)]
    B = s.rhs(directions=dirs)
    assert B.shape == (s.layout.size, 64)
    res = s.gmres(B, "bsp", tol=1e-6, maxit=1000)
    assert all(res.converged)
    X = res.solution
    # column k = 8 is config 2's angle: the reference golden
    G = golden("cfg2")
    assert abs(res.iterations[8] - int(G["gm_iters"])) <= 1
    assert relerr(X[:, 8], G["gm_x"]) < 1e-8
    # other angles against the accurate oracle (dense Schur maps)
    prob, lat = oracle_problem(c)
    itf = Interface(prob, lat, backend="schur")
    pc = Preconditioner(itf, "bsp")
    for k in (0, 21, 63):
        home, tr = lifting_traces(prob, lat, [dirs[k]])
        b = np.zeros(itf.size, complex)
        for f, j in lat.faces[home]:
            b[itf.block(lat.m_index(j, home))] = tr[f][:, 0]
        assert relerr(B[:, k], b) < 1e-11
        ref = gmres(itf.apply_A, pc, b, tol=1e-6, maxit=1000)
        assert abs(res.iterations[k] - ref.iterations) <= 1
        assert relerr(X[:, k], ref.x) < 1e-8
