"""cfg2 block-count sweep against the reference, RHS batches of any size, and
per-preconditioner configurations.

BASELINE config 2 varies the BSP block count p over 1, 2, 4, 8 (windows:
indexing.py:158-179 for the reference rule, SURVEY.md §8d rules (ii)/(iii)
otherwise).  tests/golden/cfg2.npz carries, per p, the BSP apply of the
seeded r and the full GMRES run, every S application done by the reference's
own `restricted_apply` / `apply_interface_operator` (tests/golden/refpar.py,
`make_golden.py --cfg2-sweep`).  Tolerances: apply 1e-10 (reference SuperLU
floor on the scatterer subdomain), GMRES iterations +-1 (exact
expected), x 1e-8 (BASELINE north_star), histories 1e-8 relative.
"""

import math

import numpy as np
import pytest

from conftest import cvec, golden, product_problem, relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200 import krylov, preconditioner  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS  # noqa: E402
from paper_2209_10886_b200.interface_system import GmresOptions, GpuInterfaceSystem, SweepConfig  # noqa: E402

_S = {}


def cfg2(fused=True):
    if fused not in _S:
        spec, part = product_problem(CONFIGS[2])
        _S[fused] = GpuInterfaceSystem(spec, part, fused=fused)
    return _S[fused]


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_cfg2_bsp_apply_per_block_count(p, fused):
    G = golden("cfg2")
    if f"M_bsp_p{p}" not in G.files:
        pytest.skip("cfg2 golden without the block sweep (make_golden.py --cfg2-sweep)")
    s = cfg2(fused)
    s.configure(SweepConfig(blocks=p))
    assert relerr(s.bsp_apply(G["r"]), G[f"M_bsp_p{p}"]) < 1e-10


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_cfg2_gmres_per_block_count(p):
    G = golden("cfg2")
    if f"gm_iters_p{p}" not in G.files:
        pytest.skip("cfg2 golden without the block sweep (make_golden.py --cfg2-sweep)")
    s = cfg2()
    s.configure(SweepConfig(blocks=p))
    res = s.gmres(G["b"], "bsp", tol=1e-6, maxit=1000)
    want = int(G[f"gm_iters_p{p}"])
    assert abs(res.iterations - want) <= 1, (p, res.iterations, want)
    assert res.converged
    assert relerr(res.solution, G[f"gm_x_p{p}"]) < 1e-8
    h = np.asarray(G[f"gm_hist_p{p}"])
    n = min(len(res.history), len(h))
    np.testing.assert_allclose(res.history[:n], h[:n], rtol=1e-8, atol=1e-14)
    assert relerr(s.apply_interface_operator(res.solution), G["b"]) < 1e-6


@pytest.mark.parametrize("R", [3, 5, 7])
def test_gmres_any_rhs_count(R):
    """Batched GMRES takes any number of right-hand sides (no power-of-two
    restriction): each column equals its own single-RHS solve."""
    c = CONFIGS[1]
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part)
    dirs = [(math.cos(t), math.sin(t)) for t in np.linspace(0.1, 2.0, R)]
    B = s.rhs(directions=dirs)
    res = s.gmres(B, "bsp", tol=1e-6, maxit=200)
    assert all(res.converged)
    for r in range(R):
        one = s.gmres(np.ascontiguousarray(B[:, r]), "bsp", tol=1e-6, maxit=200)
        assert res.iterations[r] == one.iterations
        assert relerr(res.solution[:, r], one.solution) < 1e-12
        np.testing.assert_allclose(res.history[r], one.history, rtol=1e-10, atol=1e-15)


def test_preconditioners_keep_their_configuration():
    """step_schedule() leaves the system's configuration alone, and
    preconditioners built for different block counts coexist (each call and
    each krylov.gmres runs under the preconditioner's own windows)."""
    G = golden("cfg2")
    s = cfg2()
    base = SweepConfig(blocks=4)
    s.configure(base)
    recs = preconditioner.step_schedule(SweepConfig(kind="sp"), s)
    assert len(recs) == 2 * (s.partition.n_groups - 1)
    assert s.sweep == base
    m1 = preconditioner.make_preconditioner(s, SweepConfig(blocks=1))
    m8 = preconditioner.make_preconditioner(s, SweepConfig(blocks=8))
    assert s.sweep == base
    r = G["r"]
    if "M_bsp_p8" in G.files:
        assert relerr(m8(r), G["M_bsp_p8"]) < 1e-10
    assert relerr(m1(r), G["M_bsp1"]) < 1e-10
    assert s.sweep == base
    res = krylov.gmres(s.apply_interface_operator, m8, G["b"], GmresOptions(tol=1e-6, maxit=1000))
    if "gm_iters_p8" in G.files:
        assert abs(res.iterations - int(G["gm_iters_p8"])) <= 1
        assert relerr(res.solution, G["gm_x_p8"]) < 1e-8
    assert s.sweep == base
