"""GPU: `krylov.gmres(apply_A, apply_M, b, opts)` with arbitrary linear
callables (SPEC.md:399-407 examples): the generic path runs the fast path's
algorithm with the Krylov basis on the GPU and gives the same iterations and
solution as the library's hs_gmres on the same operators."""

import numpy as np
import pytest

from conftest import cvec, golden, product_problem, relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200 import krylov  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS  # noqa: E402
from paper_2209_10886_b200.interface_system import GmresOptions, GpuInterfaceSystem, SweepConfig  # noqa: E402


def test_identity_one_iteration():
    b = cvec(1, 40)
    r = krylov.gmres(lambda x: x, None, b, GmresOptions(tol=1e-12))
    assert r.iterations == 1 and r.converged
    assert relerr(r.solution, b) < 1e-15


def test_zero_rhs():
    r = krylov.gmres(lambda x: 2 * x, None, np.zeros(10, complex))
    assert r.iterations == 0 and r.converged and np.all(r.solution == 0)


def test_dense_50x50_vs_direct():
    """random dense complex 50x50 well-conditioned system ->
    ||x - x_direct|| / ||x_direct|| <= 1e-8 at tol 1e-10."""
    rng = np.random.default_rng(3)
    A = np.eye(50) * 6 + (rng.standard_normal((50, 50)) + 1j * rng.standard_normal((50, 50))) / 5
    b = cvec(4, 50)
    r = krylov.gmres(lambda x: A @ x, None, b, GmresOptions(tol=1e-10, maxit=100))
    assert r.converged
    assert relerr(r.solution, np.linalg.solve(A, b)) <= 1e-8
    assert np.all(np.diff(r.history) <= 1e-12)
    # right preconditioning with an approximate inverse
    Minv = np.linalg.inv(A + 0.1 * np.eye(50))
    rp = krylov.gmres(lambda x: A @ x, lambda x: Minv @ x, b, GmresOptions(tol=1e-10, maxit=100))
    assert rp.converged and rp.iterations < r.iterations
    assert relerr(rp.solution, np.linalg.solve(A, b)) <= 1e-8


@pytest.mark.parametrize("k", [1, 2])
def test_wrapped_system_operators_match_fast_path(k):
    """The system's own operators wrapped in lambdas take the generic path:
    same iterations, same solution, same history."""
    c = CONFIGS[k]
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
    G = golden(f"cfg{k}")
    fast = krylov.gmres(s.apply_interface_operator, s.bsp_apply, G["b"], GmresOptions(tol=1e-6, maxit=1000))
    gen = krylov.gmres(lambda x: s.apply_interface_operator(x), lambda x: s.bsp_apply(x), G["b"],
                       GmresOptions(tol=1e-6, maxit=1000))
    assert gen.iterations == fast.iterations == int(G["gm_iters"])
    assert relerr(gen.solution, fast.solution) < 1e-11
    assert relerr(gen.solution, G["gm_x"]) < 1e-8
    np.testing.assert_allclose(gen.history, fast.history, rtol=1e-10)
    # torch vectors in, torch vectors out
    bt = torch.from_numpy(np.asarray(G["b"])).cuda()
    gt = krylov.gmres(lambda x: s.apply_interface_operator(x), lambda x: s.bsp_apply(x), bt,
                      GmresOptions(tol=1e-6, maxit=1000))
    assert isinstance(gt.solution, torch.Tensor) and gt.solution.is_cuda
    assert relerr(gt.solution.cpu().numpy(), fast.solution) < 1e-11
