"""GPU: field reconstruction and the end-to-end driver.

Acceptance criteria 4 and 9 of SPEC.md:528-538 on the GPU path: the stitched
domain-decomposition field matches the mono-domain solve (CPU oracle restating
discretization.py:335-370, and the reference's own mono field for cfg1).
"""

import numpy as np
import pytest

from conftest import golden, oracle_problem, product_problem, relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200.configs import CONFIGS, small_case  # noqa: E402
from paper_2209_10886_b200.driver import compare_with_mono, solve_problem  # noqa: E402
from paper_2209_10886_b200.interface_system import GmresOptions, GpuInterfaceSystem, SweepConfig  # noqa: E402


@pytest.mark.parametrize("n1,n2", [(2, 2), (3, 2)])
def test_mono_equivalence(n1, n2):
    from oracle.fd import mono_solve
    c = small_case(n1, n2, 20)
    spec, part = product_problem(c)
    prob, lat = oracle_problem(c)
    mono = mono_solve(prob, lat)
    rep = solve_problem(spec, part, SweepConfig(kind="sp"), GmresOptions(tol=1e-10, maxit=500),
                        run_mono_check=True, mono=mono)
    assert rep.converged
    assert rep.error_vs_mono["max_rel"] <= 1e-8
    assert rep.steps_per_iteration == 2 * (n1 + n2 - 2)


def test_degenerate_1x1():
    from oracle.fd import mono_solve
    c = small_case(1, 1, 8)
    spec, part = product_problem(c)
    prob, lat = oracle_problem(c)
    rep = solve_problem(spec, part, SweepConfig(kind="sp"), GmresOptions(tol=1e-10), mono=mono_solve(prob, lat))
    assert rep.iterations == 0
    assert rep.error_vs_mono["max_rel"] <= 1e-13


def test_cfg1_field_vs_oracle_and_reference_mono():
    from oracle import Interface
    from oracle.pipeline import reconstruct
    c = CONFIGS[1]
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part)
    res = s.gmres(s.rhs(), "bsp", tol=1e-10, maxit=1000)
    assert res.converged
    field = s.reconstruct_solution(res.solution)
    prob, lat = oracle_problem(c)
    itf = Interface(prob, lat)
    ref = reconstruct(itf, res.solution, itf.liftings())
    assert relerr(field, ref) < 1e-10  # reference SuperLU floor on the scatterer subdomain
    G = golden("cfg1")
    err = compare_with_mono(field, G["mono"])
    assert err["max_rel"] < 1e-7


def test_linearity_and_zero():
    c = small_case(3, 3, 16)
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part)
    rng = np.random.default_rng(4)
    L = s.layout.size
    g1 = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    g2 = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    a, b = 0.5 - 2j, 1.5 + 0.25j
    f = s.reconstruct_solution(a * g1 + b * g2, with_lifting=False)
    f12 = a * s.reconstruct_solution(g1, with_lifting=False) + b * s.reconstruct_solution(g2, with_lifting=False)
    assert relerr(f, f12) < 1e-12
    assert not np.any(s.reconstruct_solution(np.zeros(L, complex), with_lifting=False))


def test_reconstruction_vs_oracle_local_solves():
    from oracle import Interface
    from oracle.pipeline import reconstruct
    c = small_case(3, 2, 16)
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part)
    prob, lat = oracle_problem(c)
    itf = Interface(prob, lat)
    rng = np.random.default_rng(5)
    g = rng.standard_normal(itf.size) + 1j * rng.standard_normal(itf.size)
    assert relerr(s.reconstruct_solution(g), reconstruct(itf, g, itf.liftings())) < 1e-11


def test_convergence_trend_acceptance_6():
    """SPEC acceptance 6 on the GPU path: kappa = 2 pi, n = 25, N1 = 5,
    N2 in {5, 10}: SP and BSP converge to 1e-6, BSP needs at least SP's
    iterations, and fewer total sequential steps at N2 = 10; the iteration
    counts equal the CPU oracle's."""
    from oracle.pipeline import solve_problem as oracle_solve
    out = {}
    for n2 in (5, 10):
        c = small_case(5, n2, 25)
        spec, part = product_problem(c)
        prob, lat = oracle_problem(c)
        for kind in ("sp", "bsp"):
            rep = solve_problem(spec, part, SweepConfig(kind=kind), GmresOptions(tol=1e-6, maxit=500),
                                reconstruct=False)
            assert rep.converged
            ref = oracle_solve(prob, lat, kind=kind, tol=1e-6, maxit=500)
            assert abs(rep.iterations - ref.iterations) <= 1, (n2, kind, rep.iterations, ref.iterations)
            out[(n2, kind)] = (rep.iterations, rep.steps_per_iteration)
    for n2 in (5, 10):
        assert out[(n2, "bsp")][0] >= out[(n2, "sp")][0]
    sp, bsp = out[(10, "sp")], out[(10, "bsp")]
    assert bsp[0] * bsp[1] <= sp[0] * sp[1]
