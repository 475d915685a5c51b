"""GPU: the peer-memory all-reduce of the sharded Arnoldi (SURVEY.md §8f #3:
the inner products of the row-band GMRES without an NCCL call; PAPER.md:339
row ranks).  G ranks are emulated by G co-resident CTAs on one GPU (the
multi-GPU form runs the same kernel, one CTA per GPU over the CUDA-IPC
mappings); every CTA runs all reductions back to back inside one launch, so a
fast rank races into the next epoch while the others still read the current
one -- the parity buffers + consumed counters must keep every result exact:
each rank holds bitwise the rank-order sum of the G partials."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from conftest import product_problem  # noqa: E402
from paper_2209_10886_b200.configs import small_case  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem  # noqa: E402

_S = []


def ctx():
    if not _S:
        spec, part = product_problem(small_case(2, 2, 8))
        _S.append(GpuInterfaceSystem(spec, part))
    return _S[0].ctx


@pytest.mark.parametrize("G,count,repeats", [(2, 1, 50), (2, 138, 200), (4, 70, 100), (8, 4096, 20), (3, 999, 64)])
def test_peer_allreduce_emulated(G, count, repeats):
    rng = np.random.default_rng(G * 1000 + count)
    x = rng.standard_normal((repeats, G, count)) * 10.0 ** rng.integers(-8, 8, (repeats, G, count))
    out = np.empty_like(x)
    ctx().call("hs_test_peer_allreduce", G, count, repeats, C.c_void_p(x.ctypes.data), C.c_void_p(out.ctypes.data))
    want = np.zeros((repeats, count))
    for g in range(G):  # rank order 0 .. G-1, the kernel's additions
        want = want + x[:, g, :]
    for g in range(G):
        assert np.array_equal(out[:, g, :], want), (g, np.abs(out[:, g, :] - want).max())


def test_peer_allreduce_rejects_bad_sizes():
    x = np.zeros(10)
    with pytest.raises(ValueError):
        ctx().call("hs_test_peer_allreduce", 9, 1, 1, C.c_void_p(x.ctypes.data), C.c_void_p(x.ctypes.data))
    with pytest.raises(ValueError):
        ctx().call("hs_test_peer_allreduce", 2, 5000, 1, C.c_void_p(x.ctypes.data), C.c_void_p(x.ctypes.data))
