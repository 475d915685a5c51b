"""ctypes binding of libhsb200.so (include/hsb200.h).

There is no fallback: if the library is missing the import of this module
raises, and every GPU entry point of the package goes through it.
Return codes map to the reference's exception types: > 0 -> ValueError
(interface_system.py:58-62, discretization.py:176-181, 280-291), < 0 ->
RuntimeError (discretization.py:171-174).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HS_LIB=debug: the device-checks build (bounds asserts + spin watchdogs,
# include/hsb200.h hs_debug_check); same ABI, same arithmetic
LIB_PATH = os.path.join(_HERE, "_lib", "libhsb200_debug.so" if os.environ.get("HS_LIB") == "debug" else "libhsb200.so")

HS_MEM_HOST, HS_MEM_DEVICE = 0, 1
HS_APPLY_S, HS_APPLY_IMS = 0, 1
HS_PC_NONE, HS_PC_SP, HS_PC_BSP = 0, 1, 2
HS_SEAM_DEDUP, HS_SEAM_LITERAL = 0, 1

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2209_10886_b200._build` "
        "(there is no CPU fallback)")

lib = C.CDLL(LIB_PATH)

_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_pI32 = C.POINTER(C.c_int32)

_SIGS = {
    "hs_version": (C.c_char_p, []),
    "hs_last_error": (C.c_char_p, [_P]),
    "hs_create": (_I, [C.POINTER(_P), _I, _I, _I, _I, _D, _D, _D, _D, _I, _I]),
    "hs_destroy": (_I, [_P]),
    "hs_set_dirichlet": (_I, [_P, _I, _I, _pI32, _I]),
    "hs_factor": (_I, [_P]),
    "hs_lifting_rhs": (_I, [_P, _P, _I, _P, _I]),
    "hs_apply": (_I, [_P, _I, _P, _P, _I, _I]),
    "hs_reconstruct": (_I, [_P, _P, _P, _P, _I]),
    "hs_restricted_apply": (_I, [_P, _P, _P, _I, _pI32, _I, _pI32, _I, _I]),
    "hs_set_windows": (_I, [_P, _I, _pI32, _pI32, _I]),
    "hs_set_precond_options": (_I, [_P, _I, _I]),
    "hs_precond": (_I, [_P, _I, _P, _P, _I, _I]),
    "hs_half_apply": (_I, [_P, _I, _P, _P, _I, _I]),
    "hs_gmres": (_I, [_P, _I, _P, _P, _I, _D, _I, _pI32, C.POINTER(_D), _pI32, _I]),
    "hs_sizes": (_I, [_P, C.POINTER(C.c_int64), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    "hs_pairs": (_I, [_P, _pI32]),
    "hs_block_owner": (_I, [_P, _pI32]),
    "hs_schedule": (_I, [_P, _I, _pI32, _I, C.POINTER(_I)]),
    "hs_exchange_plan": (_I, [_P, _I, _I, _I, _pI32, _I, C.POINTER(_I)]),
    "hs_get_schur": (_I, [_P, _I, _I, _P]),
    "hs_gmres_basis": (_I, [_P, _P, _I, C.POINTER(_I)]),
    "hs_test_peer_allreduce": (_I, [_P, _I, _I, _I, _P, _P]),
    "hs_debug_check": (_I, [_P, C.POINTER(C.c_uint64), C.POINTER(_I)]),
    "hs_debug_selftest": (_I, [_P]),
    "hs_set_schur": (_I, [_P, _I, _I, _P]),
    "hs_set_async": (_I, [_P, _I]),
    "hs_sync": (_I, [_P]),
    "hs_stream": (_I, [_P, C.POINTER(C.c_uint64)]),
    "hs_set_kernel_timing": (_I, [_P, _I]),
    "hs_kernel_stats": (_I, [_P, C.POINTER(C.c_int64), C.POINTER(_D), C.POINTER(_D), C.POINTER(_D), _I]),
    "hs_set_map_mode": (_I, [_P, _I]),
    "hs_set_gmres_mode": (_I, [_P, _I]),
    "hs_set_emulated_ranks": (_I, [_P, _I]),
    "hs_set_trace": (_I, [_P, _I]),
    "hs_peer_export": (_I, [_P, C.POINTER(C.c_uint8)]),
    "hs_peer_open": (_I, [_P, C.POINTER(C.c_uint8), _I]),
    "hs_fused_plan": (_I, [_P, _I, _I, C.POINTER(C.c_int32), _I, C.POINTER(_I)]),
    "hs_map_once_plan": (_I, [_P, _I, C.POINTER(C.c_int32), _I, C.POINTER(_I)]),
    "hs_precond_batch": (_I, [_P, _I, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _I, _I]),
    "hs_get_trace": (_I, [_P, C.POINTER(C.c_uint64), _I, C.POINTER(_I)]),
    "hs_set_fused": (_I, [_P, _I]),
    "hs_memory": (_I, [_P, C.POINTER(C.c_int64)]),
    "hs_launch_count": (_I, [_P, C.POINTER(C.c_int64)]),
    "hs_nccl_unique_id": (_I, [C.POINTER(C.c_uint8)]),
    "hs_comm_init": (_I, [_P, C.POINTER(C.c_uint8)]),
}

EXPORTS = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def version() -> str:
    return lib.hs_version().decode()


def check(rc: int, ctx=None):
    if rc == 0:
        return
    msg = (lib.hs_last_error(ctx) or b"").decode()
    if rc > 0:
        raise ValueError(msg or f"hsb200 error {rc}")
    raise RuntimeError(msg or f"hsb200 error {rc}")


def i32(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(list(seq) if not isinstance(seq, np.ndarray) else seq, dtype=np.int32))


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_pI32)


class Context:
    """Owning handle of one hs_ctx (one GPU, or plan-only with device=-1)."""

    def __init__(self, device: int, n1: int, n2: int, n: int, h: float, kappa: float, tau: complex,
                 rank: int = 0, nranks: int = 1):
        self.h_ = _P()
        tau = complex(tau)
        check(lib.hs_create(C.byref(self.h_), int(device), int(n1), int(n2), int(n), float(h), float(kappa),
                            tau.real, tau.imag, int(rank), int(nranks)), None)
        self.device = device
        L = C.c_int64()
        nsub, ng, npairs = _I(), _I(), _I()
        lib.hs_sizes(self.h_, C.byref(L), C.byref(nsub), C.byref(ng), C.byref(npairs))
        self.L, self.nsub, self.ngroups, self.npairs = L.value, nsub.value, ng.value, npairs.value

    def __del__(self, _destroy=lib.hs_destroy):  # bound at definition: module globals may be gone at exit
        h = getattr(self, "h_", None)
        if h is not None and h.value:
            self.h_ = None
            try:
                _destroy(h)
            except (TypeError, AttributeError):  # interpreter teardown: the process is exiting anyway
                pass

    def close(self):
        self.__del__()

    def call(self, name, *args):
        rc = getattr(lib, name)(self.h_, *args)
        check(rc, self.h_)
        return rc

    # ---- introspection
    def pairs(self) -> np.ndarray:
        out = np.zeros((self.npairs, 4), dtype=np.int32)
        self.call("hs_pairs", iptr(out))
        return out

    def block_owner(self) -> np.ndarray:
        out = np.zeros(self.npairs, dtype=np.int32)
        self.call("hs_block_owner", iptr(out))
        return out

    def schedule(self, kind: int) -> np.ndarray:
        cnt = _I()
        self.call("hs_schedule", int(kind), None, 0, C.byref(cnt))
        out = np.zeros((max(cnt.value, 1), 3), dtype=np.int32)
        self.call("hs_schedule", int(kind), iptr(out), cnt.value, C.byref(cnt))
        return out[:cnt.value]

    def exchange_plan(self, kind: int, peer: int, recv: bool = False) -> np.ndarray:
        """(step, block, slot) triples sent to / received from `peer`."""
        cnt = _I()
        self.call("hs_exchange_plan", int(kind), int(peer), int(recv), None, 0, C.byref(cnt))
        out = np.zeros((max(cnt.value, 1), 3), dtype=np.int32)
        self.call("hs_exchange_plan", int(kind), int(peer), int(recv), iptr(out), cnt.value, C.byref(cnt))
        return out[:cnt.value]

    def stream(self) -> int:
        s = C.c_uint64()
        self.call("hs_stream", C.byref(s))
        return s.value

    def kernel_stats(self, reset: bool = False):
        """(launches, ms, algorithmic bytes, algorithmic flops) of the step kernels."""
        n, ms, by, fl = C.c_int64(), _D(), _D(), _D()
        self.call("hs_kernel_stats", C.byref(n), C.byref(ms), C.byref(by), C.byref(fl), int(reset))
        return n.value, ms.value, by.value, fl.value

    def launches(self) -> int:
        v = C.c_int64()
        self.call("hs_launch_count", C.byref(v))
        return v.value

    def memory(self) -> int:
        b = C.c_int64()
        self.call("hs_memory", C.byref(b))
        return b.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib.hs_nccl_unique_id(buf))
    return bytes(buf)
