"""GPU: device-memory accounting of a context (hs_memory) and no leaks.

hs_memory reports the live device allocations of one context; repeated
applies / GMRES solves / refactorisations must not grow it, and destroying the
context must return the memory to the device.
"""

import gc

import pytest

from conftest import cvec, product_problem

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200.configs import small_case  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402


def _free():
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


def test_memory_stable_and_released():
    c = small_case(4, 3, 24)
    spec, part = product_problem(c)
    free0 = _free()
    sys_ = GpuInterfaceSystem(spec, part, sweep=SweepConfig(kind="bsp"))
    L = sys_.layout.size
    n = spec.cells_per_side
    maps = 12 * 16 * (2 * n) ** 2  # lower bound: every subdomain's compact map has >= 2 faces
    b = sys_.rhs()
    sys_.apply_interface_operator(cvec(1, L))
    sys_.precondition(cvec(2, L))
    res = sys_.gmres(b, tol=1e-8, maxit=200)
    assert res.converged
    m1 = sys_.ctx.memory()
    assert m1 > 0 and m1 >= maps
    # steady state: the same calls again allocate nothing new
    for _ in range(3):
        sys_.apply_interface_operator(cvec(3, L))
        sys_.precondition(cvec(4, L))
        sys_.gmres(b, tol=1e-8, maxit=200)
    assert sys_.ctx.memory() == m1
    # a second factorisation replaces, not adds to, the factors and maps
    sys_.ctx.call("hs_factor")
    assert sys_.ctx.memory() <= m1
    res2 = sys_.gmres(b, tol=1e-8, maxit=200)
    assert res2.iterations == res.iterations
    # the accounting matches what the device lost (within allocator granularity)
    used = free0 - _free()
    assert used >= 0.9 * sys_.ctx.memory() - (64 << 20)
    sys_.close()
    with pytest.raises(ValueError):  # a closed system refuses calls
        sys_.apply_interface_operator(cvec(3, L))
    del sys_
    gc.collect()
    assert free0 - _free() <= (64 << 20)
