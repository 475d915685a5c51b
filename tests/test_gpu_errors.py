"""GPU: the C ABI rejects bad calls with ValueError (user error) and never
crashes or corrupts the context (SURVEY.md §8b error behaviour: >0 user error
-> ValueError, <0 CUDA/NCCL/singular -> RuntimeError)."""

import ctypes as C

import numpy as np
import pytest

from conftest import cvec, product_problem

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2209_10886_b200 import native  # noqa: E402
from paper_2209_10886_b200.configs import small_case  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402


@pytest.fixture(scope="module")
def system():
    spec, part = product_problem(small_case(3, 3, 16))
    return GpuInterfaceSystem(spec, part, sweep=SweepConfig(kind="bsp"))


def test_bad_vector_shapes(system):
    L = system.layout.size
    with pytest.raises(ValueError):
        system.apply_interface_operator(np.zeros(L + 1, dtype=np.complex128))
    with pytest.raises(ValueError):
        system.bsp_apply(np.zeros((L, 3, 2), dtype=np.complex128))


def test_bad_abi_arguments(system):
    ctx = system.ctx
    L = system.layout.size
    g = np.ascontiguousarray(cvec(1, L))
    out = np.empty_like(g)
    p_in, p_out = C.c_void_p(g.ctypes.data), C.c_void_p(out.ctypes.data)
    with pytest.raises(ValueError):  # nrhs out of range
        ctx.call("hs_apply", native.HS_APPLY_S, p_in, p_out, 0, native.HS_MEM_HOST)
    with pytest.raises(ValueError):
        ctx.call("hs_apply", native.HS_APPLY_S, p_in, p_out, 2048, native.HS_MEM_HOST)
    with pytest.raises(ValueError):  # unknown memory kind
        ctx.call("hs_apply", native.HS_APPLY_S, p_in, p_out, 1, 7)
    with pytest.raises(ValueError):  # unknown preconditioner kind
        ctx.call("hs_precond", 9, p_in, p_out, 1, native.HS_MEM_HOST)
    with pytest.raises(ValueError):  # GMRES tolerance / maxit
        ctx.call("hs_gmres", native.HS_PC_BSP, p_in, p_out, 1, 0.0, 10, None, None, None, native.HS_MEM_HOST)
    with pytest.raises(ValueError):
        ctx.call("hs_gmres", native.HS_PC_BSP, p_in, p_out, 1, 1e-6, 0, None, None, None, native.HS_MEM_HOST)
    with pytest.raises(ValueError):  # Dirichlet cell out of range
        cells = np.array([10 ** 6], dtype=np.int32)
        ctx.call("hs_set_dirichlet", 1, 1, native.iptr(cells), 1)
    with pytest.raises(ValueError):  # subdomain out of range
        ctx.call("hs_set_dirichlet", 9, 1, None, 0)
    # the context still works after all of that
    ref = system.apply_interface_operator(g)
    assert np.isfinite(ref).all()


def test_unfactored_context_refuses():
    ctx = native.Context(0, 2, 2, 8, 0.1, 3.0, 3j)
    g = np.zeros(ctx.L, dtype=np.complex128)
    out = np.empty_like(g)
    with pytest.raises(ValueError):
        ctx.call("hs_apply", native.HS_APPLY_S, C.c_void_p(g.ctypes.data), C.c_void_p(out.ctypes.data), 1,
                 native.HS_MEM_HOST)
    ctx.close()


def test_plan_only_context_cannot_run_kernels():
    ctx = native.Context(-1, 2, 2, 8, 0.1, 3.0, 3j)
    with pytest.raises(ValueError):
        ctx.call("hs_factor")
    ctx.close()
