"""GPU: the FP64 DMMA contraction paths.

* multi-RHS with per-subdomain maps (K4): every column equals the single-RHS
  HBM kernel's result;
* shared-operator mode (class maps, one contraction per step): equals the
  per-subdomain mode on every entry point (the maps are the same numbers,
  discretization.py:224-229), and GMRES takes the same iterations;
* shared mode refuses n not divisible by the 16-wide K chunk.
"""

import numpy as np
import pytest

from conftest import cvec, golden, product_problem, relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200.configs import CONFIGS, small_case  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

_S = {}


def system(k, maps):
    key = (k, maps)
    if key not in _S:
        if k >= 3:
            for kk in [x for x in _S if x[0] >= 3 and x != key]:
                del _S[kk]
        c = CONFIGS[k] if isinstance(k, int) else k
        spec, part = product_problem(c)
        _S[key] = GpuInterfaceSystem(spec, part, maps=maps, sweep=SweepConfig(blocks=c["blocks"]))
    return _S[key]


@pytest.mark.parametrize("k,R", [(1, 40), (2, 40), (2, 16), (2, 64), (2, 100), (2, 128)])
def test_multi_rhs_dmma_equals_single(k, R):
    """R <= 32: 32-column tasks; R > 32: 64-column tasks (k_zmma2), partial
    last chunks for R = 40, 100."""
    s = system(k, "subdomain")
    L = s.layout.size
    X = cvec(3, L, R)
    Y = s.apply_interface_operator(X)
    Z = s.bsp_apply(X)
    for r in sorted({0, R // 2, 31 % R, min(32, R - 1), R - 1}):
        x = np.ascontiguousarray(X[:, r])
        assert relerr(Y[:, r], s.apply_interface_operator(x)) < 1e-14
        assert relerr(Z[:, r], s.bsp_apply(x)) < 1e-13


@pytest.mark.parametrize("k", [1, 2, 3])
def test_shared_mode_equals_subdomain_mode(k):
    a, b = system(k, "subdomain"), system(k, "shared")
    L = a.layout.size
    g = cvec(9, L)
    assert relerr(b.apply_scattering(g), a.apply_scattering(g)) < 1e-14
    assert relerr(b.apply_interface_operator(g), a.apply_interface_operator(g)) < 1e-14
    assert relerr(b.bsp_apply(g), a.bsp_apply(g)) < 1e-13
    assert relerr(b.sgs_apply(g), a.sgs_apply(g)) < 1e-13
    ng = a.partition.n_groups
    assert relerr(b.restricted_apply(g, {ng // 2}, {ng // 2 + 1}), a.restricted_apply(g, {ng // 2}, {ng // 2 + 1})) < 1e-14
    G = [(s.i1, s.i2) for s in a.partition.subdomains[:3]] + [tuple(a.home)]
    for sub in G:
        assert np.array_equal(b.schur_map(sub), a.schur_map(sub))
    rb = b.rhs()
    assert relerr(rb, a.rhs()) < 1e-15
    ra, rs = a.gmres(rb, "bsp", tol=1e-6, maxit=1000), b.gmres(rb, "bsp", tol=1e-6, maxit=1000)
    assert ra.iterations == rs.iterations and rs.converged
    assert relerr(rs.solution, ra.solution) < 1e-10


def test_shared_mode_vs_reference_golden_cfg2():
    G = golden("cfg2")
    s = system(2, "shared")
    assert relerr(s.apply_interface_operator(G["g"]), G["Ag"]) < 1e-10
    assert relerr(s.bsp_apply(G["r"]), G["M_bsp"]) < 1e-10
    res = s.gmres(G["b"], "bsp", tol=1e-6, maxit=1000)
    assert res.iterations == int(G["gm_iters"])
    assert relerr(res.solution, G["gm_x"]) < 1e-8


def test_shared_mode_cfg5_vs_reference_golden():
    """Shared class maps + DMMA at the headline config against the reference
    golden (tests/golden/cfg5.npz) and the accurate oracle (see
    test_gpu_scale.test_cfg5_vs_reference_golden for the floors)."""
    G = golden("cfg5")
    s = system(5, "shared")
    L = s.layout.size
    r = cvec(int(G["seed_r"]), L)
    z = s.bsp_apply(r)
    assert relerr(z, G["M_bsp8"]) < 2e-9
    assert relerr(z, G["M_bsp8"] + G["acc_dbsp"]) < 1e-12
    res = s.gmres(G["b"], "bsp", tol=1e-6, maxit=1000)
    assert res.converged and abs(res.iterations - int(G["gm_iters"])) <= 1, res.iterations
    assert relerr(res.solution, G["gm_x"]) < 1e-8
    assert relerr(res.solution, G["gm_x"] + G["acc_dx"]) < 1e-11
    assert relerr(s.apply_interface_operator(res.solution), G["b"]) < 1e-6


def test_shared_mode_needs_n_multiple_of_32():
    spec, part = product_problem(small_case(2, 2, 8))
    with pytest.raises(ValueError):
        GpuInterfaceSystem(spec, part, maps="shared")


@pytest.mark.parametrize("k", [1, 2, 3])
def test_hostloop_mgs_equals_cooperative(k):
    """The sharded Arnoldi (host-driven MGS over owned blocks, the algorithm run
    across row bands with one allreduce per inner product) on one GPU."""
    s = system(k, "subdomain")
    b = s.rhs()
    a = s.gmres(b, "bsp", tol=1e-6, maxit=1000, arnoldi="auto")
    for mode in ("hostloop", "grid"):
        h = s.gmres(b, "bsp", tol=1e-6, maxit=1000, arnoldi=mode)
        assert h.iterations == a.iterations and h.converged
        assert relerr(h.solution, a.solution) < 1e-12
        np.testing.assert_allclose(h.history, a.history, rtol=1e-10)


def test_hostloop_mgs_batched_cfg4():
    import math
    from paper_2209_10886_b200.configs import angles
    s = system(4, "subdomain")
    dirs = [(math.cos(t), math.sin(t)) for t in angles(CONFIGS[4])][:8]
    B = s.rhs(directions=dirs)
    a = s.gmres(B, "bsp", tol=1e-6, maxit=1000)
    h = s.gmres(B, "bsp", tol=1e-6, maxit=1000, arnoldi="hostloop")
    assert h.iterations == a.iterations
    assert relerr(h.solution, a.solution) < 1e-12


@pytest.mark.parametrize("k", [1, 2, 3])
def test_cgs2_arnoldi(k):
    """CGS2: iterations within +-1 of MGS, same solution to
    the GMRES tolerance, and the reference's x within 1e-8 where a golden exists."""
    s = system(k, "subdomain")
    b = s.rhs()
    a = s.gmres(b, "bsp", tol=1e-6, maxit=1000)
    c2 = s.gmres(b, "bsp", tol=1e-6, maxit=1000, arnoldi="cgs2")
    assert c2.converged and abs(c2.iterations - a.iterations) <= 1
    assert relerr(c2.solution, a.solution) < 1e-9
    assert relerr(s.apply_interface_operator(c2.solution), b) < 1e-6
    assert c2.iterations == a.iterations
    np.testing.assert_allclose(c2.history, a.history, rtol=1e-10)
