"""GPU: the fused dataflow BSP apply (one persistent launch, per-block
completion counters).  Its per-step plan (fused="steps") is bitwise identical
to the one-launch-per-step sequence, including 1-step windows (seams written
and read in the same step) and the reference-window / block-count variants;
the map-once plan (the default) equals it to rounding and matches the oracle."""

import numpy as np
import pytest

from conftest import cvec, golden, product_problem, relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200.configs import CONFIGS, small_case  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

CASES = [("small_1x4", small_case(1, 4, 8), [None, 1]), ("small_3x3", small_case(3, 3, 8), [None, 1, 2]),
         ("small_6x3", small_case(6, 3, 16), [None, 2, 5]), ("cfg1", CONFIGS[1], [None, 1, 3]),
         ("cfg2", CONFIGS[2], [None, 1, 4, 8]), ("cfg3", CONFIGS[3], [4])]


@pytest.mark.parametrize("name,c,blocks", CASES)
def test_fused_bitwise_equals_steps(name, c, blocks):
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, fused="literal")
    b = GpuInterfaceSystem(spec, part, fused="steps")
    g = cvec(13, a.layout.size)
    for p in blocks:
        a.configure(SweepConfig(blocks=p))
        b.configure(SweepConfig(blocks=p))
        za, zb = a.bsp_apply(g), b.bsp_apply(g)
        assert np.array_equal(za, zb), (name, p, relerr(zb, za))
        for _ in range(3):  # repeated launches (counter reset, ticket reuse)
            assert np.array_equal(b.bsp_apply(g), za)


def test_fused_gmres_cfg2_golden():
    G = golden("cfg2")
    spec, part = product_problem(CONFIGS[2])
    s = GpuInterfaceSystem(spec, part, fused=True)
    res = s.gmres(G["b"], "bsp", tol=1e-6, maxit=1000)
    assert res.iterations == int(G["gm_iters"])
    assert relerr(res.solution, G["gm_x"]) < 1e-8


@pytest.mark.parametrize("name,c,blocks", [("small_3x3", small_case(3, 3, 8), 2), ("small_6x3", small_case(6, 3, 16), 5),
                                           ("cfg1", CONFIGS[1], None), ("cfg2", CONFIGS[2], 4), ("cfg3", CONFIGS[3], 4)])
def test_fused_gmres_bitwise_equals_steps(name, c, blocks):
    """GMRES with A M v as ONE launch (BSP + (I - S) z, phase 3 of the fused
    per-step plan) runs bitwise the same iterations as the per-step kernels."""
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, fused="literal", sweep=SweepConfig(blocks=blocks))
    b = GpuInterfaceSystem(spec, part, fused="steps", sweep=SweepConfig(blocks=blocks))
    rhs = a.rhs() if c.get("center") is not None else cvec(5, a.layout.size)
    ra = a.gmres(rhs, "bsp", tol=1e-8, maxit=300)
    rb = b.gmres(rhs, "bsp", tol=1e-8, maxit=300)
    assert ra.iterations == rb.iterations and ra.converged and rb.converged
    assert np.array_equal(ra.solution, rb.solution), relerr(rb.solution, ra.solution)
    assert np.array_equal(np.asarray(ra.history), np.asarray(rb.history))


@pytest.mark.parametrize("name,c,R,maps", [("cfg1", CONFIGS[1], 40, "subdomain"), ("cfg2", CONFIGS[2], 64, "subdomain"),
                                           ("cfg1", CONFIGS[1], 1, "shared"), ("cfg2", CONFIGS[2], 1, "shared"),
                                           ("cfg3", CONFIGS[3], 1, "shared"), ("cfg2", CONFIGS[2], 8, "shared")])
def test_fused_dmma_equals_steps(name, c, R, maps):
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, fused=False, maps=maps, sweep=SweepConfig(blocks=c["blocks"]))
    b = GpuInterfaceSystem(spec, part, fused=11 if maps == "shared" else 3, maps=maps,
                           sweep=SweepConfig(blocks=c["blocks"]))
    g = cvec(17, a.layout.size, None if R == 1 else R)
    za = a.bsp_apply(g)
    zb = b.bsp_apply(g)
    assert relerr(zb, za) < 1e-13, relerr(zb, za)
    assert np.array_equal(b.bsp_apply(g), zb)  # the fused launch itself is deterministic


@pytest.mark.parametrize("name,c,blocks", [("small_6x3", small_case(6, 3, 16), 5), ("cfg2", CONFIGS[2], 4),
                                           ("cfg3", CONFIGS[3], 4)])
def test_host_buffer_apply_bitwise(name, c, blocks):
    """hs_precond on HOST buffers (pageable numpy, pinned torch) returns
    bitwise the device-buffer result, call after call."""
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=blocks))
    g = cvec(23, s.layout.size)
    zd = s.bsp_apply(torch.from_numpy(g).cuda()).cpu().numpy()
    zh = s.bsp_apply(g)
    assert np.array_equal(zd, zh), relerr(zh, zd)
    gp = torch.from_numpy(g).pin_memory()
    for _ in range(3):
        assert np.array_equal(s.bsp_apply(gp).numpy(), zd)


_VARIANT_SCRIPT = r"""
import hashlib, sys, numpy as np
sys.path.insert(0, 'tests')
from conftest import cvec, product_problem
from paper_2209_10886_b200.configs import CONFIGS, small_case
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
for c, blocks in ((small_case(6, 3, 16), 5), (CONFIGS[2], 4), (CONFIGS[3], 4)):
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, fused="literal", sweep=SweepConfig(blocks=blocks))
    b = GpuInterfaceSystem(spec, part, fused="steps", sweep=SweepConfig(blocks=blocks))
    g = cvec(29, a.layout.size)
    assert np.array_equal(a.bsp_apply(g), b.bsp_apply(g)), c["name"]
    m = GpuInterfaceSystem(spec, part, fused=True, sweep=SweepConfig(blocks=blocks))
    print(c["name"], hashlib.sha1(m.bsp_apply(g).tobytes()).hexdigest())
print("ok")
"""


def _run_variant(env):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT], cwd=root, env=dict(os.environ, **env),
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
    return [ln for ln in out.stdout.splitlines() if ln != "ok"]


def test_fused_variants_bitwise():
    """Every fused-kernel variant (TMA-staged, register streaming, two strips
    per tile) of the per-step plan is bitwise the per-step result, and the
    map-once plan gives bitwise the same z on the TMA-staged and the register-
    streaming kernel (one column split); the knobs are read once per process,
    so each runs in its own interpreter."""
    tma = _run_variant({"HS_FUSED_TMA": "1"})
    regs = _run_variant({"HS_FUSED_TMA": "0"})
    _run_variant({"HS_FUSED_RT": "2"})
    assert tma == regs, (tma, regs)


@pytest.mark.parametrize("name,c,blocks,ranks", [("small_6x3", small_case(6, 3, 16), 5, (2, 3)),
                                                 ("small_4x4_n160", small_case(4, 4, 160), None, (2, 4)),
                                                 ("cfg2", CONFIGS[2], 4, (2, 4, 8)), ("cfg3", CONFIGS[3], 4, (2, 8))])
@pytest.mark.parametrize("plan", [True, "steps"])
def test_emulated_row_band_ranks_bitwise(name, c, blocks, ranks, plan):
    """The multi-rank fused kernels (every block on its owner rank, output
    blocks and their counters reached in the owner's buffers -- the
    peer-memory protocol of the multi-GPU path) emulated on one GPU: bitwise
    the single-rank apply, for TMA-staged (maps <= 512 columns) and
    register-streaming (n = 160: 640 columns) kernels."""
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=blocks), fused=plan)
    g = cvec(31, s.layout.size)
    ref = s.bsp_apply(g)
    for G in ranks:
        s.ctx.call("hs_set_emulated_ranks", G)
        for _ in range(2):
            z = s.bsp_apply(g)
            assert np.array_equal(z, ref), (name, G, relerr(z, ref))
    s.ctx.call("hs_set_emulated_ranks", 1)
    assert np.array_equal(s.bsp_apply(g), ref)


MAP_ONCE_CASES = [("small_1x4", small_case(1, 4, 8), [None, 1]), ("small_5x1", small_case(5, 1, 8), [None, 1, 2]),
                  ("small_2x7_n20", small_case(2, 7, 20), [None, 1, 3]), ("small_3x3", small_case(3, 3, 8), [None, 1, 2]),
                  ("small_6x3", small_case(6, 3, 16), [None, 2, 5]), ("small_4x4_n160", small_case(4, 4, 160), [None, 3]),
                  ("cfg1", CONFIGS[1], [None, 1, 3]), ("cfg2", CONFIGS[2], [None, 1, 2, 4, 8]), ("cfg3", CONFIGS[3], [4])]


@pytest.mark.parametrize("name,c,blocks", MAP_ONCE_CASES)
def test_map_once_equals_steps(name, c, blocks):
    """The map-once plan (residual elided inside forward windows, residual and
    backward products sharing one map read) gives the step sequence's z to
    rounding, for every block count incl. 1-step windows; repeated launches are
    bitwise reproducible."""
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, fused="literal")
    b = GpuInterfaceSystem(spec, part, fused=True)
    d = GpuInterfaceSystem(spec, part, fused=False)  # per-step launches, map-once form
    g = cvec(13, a.layout.size)
    for p in blocks:
        for x in (a, b, d):
            x.configure(SweepConfig(blocks=p))
        za, zb, zd = a.bsp_apply(g), b.bsp_apply(g), d.bsp_apply(g)
        assert relerr(zb, za) < 1e-13, (name, p, relerr(zb, za))
        assert relerr(zd, za) < 1e-13, (name, p, relerr(zd, za))
        for _ in range(2):
            assert np.array_equal(b.bsp_apply(g), zb)


@pytest.mark.parametrize("name,c,blocks", [("small_1x4", small_case(1, 4, 8), 1), ("small_3x3", small_case(3, 3, 8), 2),
                                           ("small_6x3", small_case(6, 3, 16), 5), ("cfg1", CONFIGS[1], None),
                                           ("cfg2", CONFIGS[2], 8), ("cfg3", CONFIGS[3], 4)])
def test_map_once_gmres_equals_steps(name, c, blocks):
    """GMRES with A M v in map-once form -- one launch (BSP + (I - S) z reading
    each map row ~1.7 times instead of 3), and per-step launches (restricted
    residual step, (I - S) z on the upper rows + window starts): the literal
    iterations, history to 1e-8 and solution to 1e-10."""
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, fused="literal", sweep=SweepConfig(blocks=blocks))
    rhs = a.rhs() if c.get("center") is not None else cvec(5, a.layout.size)
    ra = a.gmres(rhs, "bsp", tol=1e-8, maxit=300)
    ha = np.asarray(ra.history)
    for fused in (True, False):  # one launch per A M v / per-step map-once (residual + (I - S) z rows)
        b = GpuInterfaceSystem(spec, part, fused=fused, sweep=SweepConfig(blocks=blocks))
        rb = b.gmres(rhs, "bsp", tol=1e-8, maxit=300)
        assert ra.converged and rb.converged and ra.iterations == rb.iterations, fused
        assert relerr(rb.solution, ra.solution) < 1e-10, (fused, relerr(rb.solution, ra.solution))
        hb = np.asarray(rb.history)
        assert np.max(np.abs(hb - ha) / ha) < 1e-8, fused


@pytest.mark.parametrize("name,c,blocks", [("small_6x3", small_case(6, 3, 16), 5), ("small_4x4_n160", small_case(4, 4, 160), None),
                                           ("cfg1", CONFIGS[1], None), ("cfg2", CONFIGS[2], 4), ("cfg3", CONFIGS[3], 4)])
def test_peer_memory_path_single_rank(name, c, blocks):
    """The multi-GPU peer-memory path (hs_peer_export / hs_peer_open: own
    region exported through CUDA IPC, the multi-rank kernel launched with
    self = this rank, system-scope fences) run with one rank on one GPU:
    bitwise the ordinary fused apply, and the same GMRES (A M v through the
    peer path) bit for bit."""
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=blocks))
    b = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=blocks))
    b.enable_peer_memory()
    g = cvec(37, a.layout.size)
    za = a.bsp_apply(g)
    for _ in range(2):
        zb = b.bsp_apply(g)
        assert np.array_equal(za, zb), (name, relerr(zb, za))
    rhs = a.rhs() if c.get("center") is not None else cvec(5, a.layout.size)
    ra = a.gmres(rhs, "bsp", tol=1e-8, maxit=300)
    rb = b.gmres(rhs, "bsp", tol=1e-8, maxit=300)
    assert ra.iterations == rb.iterations and np.array_equal(ra.solution, rb.solution)
    # new windows: the peer plans are rebuilt and the epoch counters restart
    for p in (2, None):
        a.configure(SweepConfig(blocks=p))
        b.configure(SweepConfig(blocks=p))
        assert np.array_equal(a.bsp_apply(g), b.bsp_apply(g)), (name, p)
    with pytest.raises(ValueError):
        b.enable_peer_memory()  # already open


@pytest.mark.parametrize("name,c,blocks", [("small_6x3", small_case(6, 3, 16), 5), ("cfg2", CONFIGS[2], 4)])
def test_precondition_batch_pipelined(name, c, blocks):
    """hs_precond_batch (host vectors copied in / out on two copy streams
    while the neighbouring vector is applied) returns bitwise the one-call
    result for every vector, numpy and pinned torch alike, for odd and even
    batch sizes and for SP as well as BSP."""
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=blocks))
    gs = [cvec(41 + i, s.layout.size) for i in range(5)]
    for kind in ("bsp", "sp"):
        ref = [s.precondition(g, kind) for g in gs]
        for nb in (1, 2, 5):
            out = s.precondition_batch(gs[:nb], kind)
            for a, b in zip(out, ref):
                assert np.array_equal(a, b), (name, kind, nb)
    pin = [torch.from_numpy(g).pin_memory() for g in gs[:3]]
    zs = [torch.empty_like(p).pin_memory() for p in pin]
    s.precondition_batch(pin, out=zs)
    for i in range(3):
        assert np.array_equal(zs[i].numpy(), s.precondition(gs[i], "bsp"))
    with pytest.raises(ValueError):
        s.precondition_batch([torch.from_numpy(gs[0]).cuda()])


@pytest.mark.parametrize("name,c,R,maps", [("small_6x3", small_case(6, 3, 16), 1, "subdomain"),
                                           ("cfg2", CONFIGS[2], 8, "subdomain"), ("cfg2", CONFIGS[2], 1, "shared"),
                                           ("cfg1", CONFIGS[1], 4, "shared")])
def test_map_once_steps_dmma_and_multi_rhs(name, c, R, maps):
    """The per-step map-once form on the DMMA contraction (R right-hand
    sides, shared class maps) and on k_step1: BSP equal to the literal step
    sequence to rounding, and batched GMRES (A M v with the (I - S) z rows of
    the map-once form) in the literal iterations."""
    spec, part = product_problem(c)
    blocks = c.get("blocks")
    a = GpuInterfaceSystem(spec, part, fused="literal", maps=maps, sweep=SweepConfig(blocks=blocks))
    d = GpuInterfaceSystem(spec, part, fused=False, maps=maps, sweep=SweepConfig(blocks=blocks))
    g = cvec(19, a.layout.size, None if R == 1 else R)
    assert relerr(d.bsp_apply(g), a.bsp_apply(g)) < 1e-13
    ra = a.gmres(g, "bsp", tol=1e-8, maxit=300)
    rd = d.gmres(g, "bsp", tol=1e-8, maxit=300)
    assert ra.iterations == rd.iterations
    assert relerr(rd.solution, ra.solution) < 1e-9


_SPLIT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, 'tests')
from conftest import cvec, product_problem, relerr
from paper_2209_10886_b200.configs import CONFIGS, small_case
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
for c, blocks in ((small_case(4, 4, 160), None), (CONFIGS[2], 4), (CONFIGS[3], 4)):
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, fused="literal", sweep=SweepConfig(blocks=blocks))
    b = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=blocks))  # map-once, split-K forced
    g = cvec(43, a.layout.size)
    za, zb = a.bsp_apply(g), b.bsp_apply(g)
    assert relerr(zb, za) < 1e-13, (c["name"], relerr(zb, za))
    for _ in range(3):  # deterministic: the pair's halves are added in half order
        assert np.array_equal(b.bsp_apply(g), zb)
    b.ctx.call("hs_set_emulated_ranks", 2)
    assert np.array_equal(b.bsp_apply(g), zb)
    b.ctx.call("hs_set_emulated_ranks", 1)
    rhs = a.rhs()
    ra, rb = a.gmres(rhs, "bsp", tol=1e-8, maxit=300), b.gmres(rhs, "bsp", tol=1e-8, maxit=300)
    assert ra.iterations == rb.iterations and relerr(rb.solution, ra.solution) < 1e-10
    p = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=blocks))
    p.enable_peer_memory()
    assert np.array_equal(p.bsp_apply(g), zb)
print("ok")
"""


def test_split_k_pairs():
    """Split-K tiles (each strip streamed by two CTAs, the second arrival adds
    the halves in half order and finishes the rows -- the large-GPU-count
    mode, forced here with HS_SPLITK=1): the literal result to rounding,
    bitwise reproducible, identical under emulated row bands and on the peer
    path, and the literal GMRES iterations."""
    out = _run_variant_script(_SPLIT_SCRIPT, {"HS_SPLITK": "1"})
    assert out.endswith("ok")


def _run_variant_script(script, env):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", script], cwd=root, env=dict(os.environ, **env),
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    return out.stdout.strip()


@pytest.mark.parametrize("name,c,blocks", [("small_6x3", small_case(6, 3, 16), 5), ("cfg1", CONFIGS[1], None),
                                           ("cfg2", CONFIGS[2], 4), ("cfg3", CONFIGS[3], 4)])
def test_kind_maps_bitwise(name, c, blocks):
    """maps="kinds" (one compact map per (operator class, face set), every
    subdomain record aliasing its kind's): bitwise the per-subdomain maps, for
    the fused apply, GMRES, the per-step path and the (I - S) apply."""
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=blocks))
    b = GpuInterfaceSystem(spec, part, maps="kinds", sweep=SweepConfig(blocks=blocks))
    assert b.ctx.memory() < a.ctx.memory() or c["n1"] * c["n2"] <= 9
    g = cvec(47, a.layout.size)
    assert np.array_equal(a.bsp_apply(g), b.bsp_apply(g))
    assert np.array_equal(a.apply_interface_operator(g), b.apply_interface_operator(g))
    rhs = a.rhs() if c.get("center") is not None else cvec(5, a.layout.size)
    ra, rb = a.gmres(rhs, "bsp", tol=1e-8, maxit=300), b.gmres(rhs, "bsp", tol=1e-8, maxit=300)
    assert ra.iterations == rb.iterations and np.array_equal(ra.solution, rb.solution)
    d = GpuInterfaceSystem(spec, part, maps="kinds", fused=False, sweep=SweepConfig(blocks=blocks))
    e = GpuInterfaceSystem(spec, part, fused=False, sweep=SweepConfig(blocks=blocks))
    assert np.array_equal(d.bsp_apply(g), e.bsp_apply(g))


_DF_VARIANT_SCRIPT = """
import numpy as np
import sys
sys.path[:0] = [".", "tests"]
from conftest import cvec, product_problem, relerr
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
for cfg, R, maps in ((2, 64, "subdomain"), (1, 40, "subdomain"), (2, 1, "shared"), (3, 1, "shared")):
    c = CONFIGS[cfg]
    spec, part = product_problem(c)
    a = GpuInterfaceSystem(spec, part, fused=False, maps=maps, sweep=SweepConfig(blocks=c["blocks"]))
    b = GpuInterfaceSystem(spec, part, fused=11 if maps == "shared" else 3, maps=maps,
                           sweep=SweepConfig(blocks=c["blocks"]))
    g = cvec(17, a.layout.size, None if R == 1 else R)
    za, zb = a.bsp_apply(g), b.bsp_apply(g)
    assert relerr(zb, za) < 1e-13, (cfg, R, maps, relerr(zb, za))
    assert np.array_equal(b.bsp_apply(g), zb)
    if maps == "shared":  # one right-hand side: GMRES runs the dataflow apply
        rhs = a.rhs()
        ra, rb = a.gmres(rhs, "bsp", tol=1e-8, maxit=300), b.gmres(rhs, "bsp", tol=1e-8, maxit=300)
        assert ra.iterations == rb.iterations and relerr(rb.solution, ra.solution) < 1e-10
print("ok")
"""


@pytest.mark.parametrize("env", [{"HS_ZMMA2_SPLIT": "1"}, {"HS_ZMMA2_DF_MO": "0"},
                                 {"HS_ZMMA2_SPLIT": "1", "HS_ZMMA2_KC64": "0"}])
def test_dmma_dataflow_variants(env):
    """k_zmma2_df variants against the per-step contraction: split-K pairs
    (HS_ZMMA2_SPLIT=1, both halves summed in half order by the later arrival),
    the full residual step instead of the map-once residual + fill tasks
    (HS_ZMMA2_DF_MO=0), the n-major shared-map form on 32-row chunks
    (HS_ZMMA2_KC64=0); apply to rounding, bitwise reproducible, GMRES
    iterations equal."""
    out = _run_variant_script(_DF_VARIANT_SCRIPT, env)
    assert out.endswith("ok")
