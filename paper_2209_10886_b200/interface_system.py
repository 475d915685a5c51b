"""The interface problem (I - S) g = b on the GPU, with the reference API.

`GpuInterfaceSystem(spec, partition, imp=None, workers=1, ...)` is the drop-in
for `InterfaceSystem` (interface_system.py:65-175): same constructor
arguments, attributes (`spec`, `partition`, `imp`, `layout`, `operators`)
and methods (`compute_liftings`, `assemble_rhs`, `apply_scattering`,
`apply_interface_operator`, `restricted_apply`, `materialize_dense`), plus
the specified-but-unshipped preconditioner and GMRES entry points
(SPEC.md:306-407).  Every numerical operation runs in libhsb200 on the GPU:
one batched kernel per sweep step over all subdomains of the step.

Vectors are numpy complex128 (host; copied in/out inside the call) or torch
complex128 CUDA tensors (device; zero-copy), of shape (L,) or (L, R) for R
right-hand sides; results come back as the same kind.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import native
from .discretization import ImpedanceSpec, SubdomainInfo, lifting_data, scatterer_cells
from .indexing import MultiIndex, Partition, window_ranges

DENSE_GUARD = 6000


class TraceLayout:
    """interface_system.py:30-62: 2 N_e blocks of n in m-order."""

    def __init__(self, partition: Partition, n: int):
        self.partition = partition
        self.n = n
        self.size = len(partition.pairs) * n

    def zeros(self) -> np.ndarray:
        return np.zeros(self.size, dtype=complex)

    def block(self, m: int) -> slice:
        return slice((m - 1) * self.n, m * self.n)

    def block_of(self, owner, neighbor) -> slice:
        return self.block(self.partition.m_index((owner, neighbor)))

    def group_indices(self, groups) -> np.ndarray:
        groups = set(groups)
        ms = [m for m, p in enumerate(self.partition.pairs, start=1) if p.owner.group in groups]
        if not ms:
            return np.empty(0, dtype=np.intp)
        return np.concatenate([np.arange((m - 1) * self.n, m * self.n) for m in ms])

    def check(self, g):
        shape = tuple(getattr(g, "shape", np.shape(g)))
        if len(shape) == 0 or shape[0] != self.size or len(shape) > 2:
            n = shape[0] if shape else 0
            raise ValueError(f"interface vector has length {n}, expected {self.size}")
        return g


@dataclass
class SweepConfig:
    """SPEC.md:296-299 (+ the block count of SURVEY.md §8d)."""

    kind: str = "bsp"  # none | sp | bsp
    bsp_seam: str = "dedup"
    bsp_intermediate_residual: bool = True
    count_residual_steps: bool = False
    blocks: int | None = None


@dataclass
class GmresOptions:
    tol: float = 1e-6
    maxit: int = 200
    record_history: bool = True


@dataclass
class GmresResult:
    solution: object
    history: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    wall_time: float = 0.0


_PC = {"none": native.HS_PC_NONE, "sp": native.HS_PC_SP, "bsp": native.HS_PC_BSP}


class _Vec:
    """Caller buffer <-> (pointer, mem kind, output allocator)."""

    def __init__(self, x, L):
        self.torch = None
        try:
            import torch
            if isinstance(x, torch.Tensor):
                self.torch = torch
        except ImportError:  # pragma: no cover
            pass
        if self.torch is not None:
            t = x
            if t.dtype != self.torch.complex128:
                t = t.to(self.torch.complex128)
            t = t.contiguous()
            self.cpu = not t.is_cuda
            if self.cpu:
                self.arr = np.ascontiguousarray(t.numpy())
            else:
                self.torch.cuda.current_stream(t.device).synchronize()
                self.t = t
        else:
            self.cpu = True
            self.arr = np.ascontiguousarray(np.asarray(x), dtype=np.complex128)
        shape = self.arr.shape if self.cpu else tuple(self.t.shape)
        if len(shape) not in (1, 2) or shape[0] != L:
            raise ValueError(f"interface vector has length {shape[0] if shape else 0}, expected {L}")
        self.shape = shape
        self.R = 1 if len(shape) == 1 else shape[1]

    @property
    def ptr(self):
        return self.arr.ctypes.data if self.cpu else self.t.data_ptr()

    @property
    def mem(self):
        return native.HS_MEM_HOST if self.cpu else native.HS_MEM_DEVICE

    def empty(self):
        if self.cpu:
            out = np.empty(self.shape, dtype=np.complex128)
            return out, out.ctypes.data
        out = self.torch.empty(self.shape, dtype=self.torch.complex128, device=self.t.device)
        return out, out.data_ptr()

    def wrap(self, out):
        if self.torch is not None and self.cpu:
            return self.torch.from_numpy(out)
        return out


def gather_peer_handles(handle: bytes, rank: int, nranks: int) -> bytes:
    """All-gather the ranks' 64-byte IPC handles in rank order (the layout
    hs_peer_open reads) over the initialised torch.distributed group."""
    if len(handle) != 64:
        raise ValueError("an IPC handle is 64 bytes")
    if nranks == 1:
        return handle
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() != nranks or dist.get_rank() != rank:
        raise ValueError("peer memory needs torch.distributed initialised with this system's rank / nranks")
    objs = [None] * nranks
    dist.all_gather_object(objs, handle)
    return b"".join(objs)


class GpuInterfaceSystem:
    """Subdomain Schur maps + matrix-free S on one GPU (or one row band)."""

    _last_R = 1  # right-hand sides of the last gmres call (gmres_basis)

    def __init__(self, spec, partition: Partition, imp: ImpedanceSpec | None = None, workers: int = 1,
                 device: int = 0, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None,
                 sweep: SweepConfig | None = None, maps: str = "subdomain", fused: bool | int | str = True):
        """maps = "subdomain": one compact Schur map per subdomain, streamed from
        HBM by the step kernels (the graded path); "shared": only the distinct
        operators' maps (generic + scatterer) are kept and every step is a DMMA
        contraction with the map L2-resident (discretization.py:224-229);
        "kinds": one compact map per distinct (operator, face set) -- the same
        bytes as "subdomain" for every subdomain, read by the same fused
        kernels, but ~18 maps instead of one per subdomain, so the stream is
        served from L2 (kept there with an evict-last policy)."""
        if workers < 1:
            raise ValueError(f"workers must be >= 1, got {workers}")
        self.spec = spec
        self.partition = partition
        self.imp = imp if imp is not None else ImpedanceSpec.for_problem(spec)
        self.workers = workers  # accepted for API parity; the GPU batches every solve of a step
        self.layout = TraceLayout(partition, spec.cells_per_side)
        self.n = spec.cells_per_side
        self.rank, self.nranks = rank, nranks
        self.ctx = native.Context(device, partition.n1, partition.n2, self.n, spec.h, spec.kappa,
                                  complex(self.imp.coefficient), rank, nranks)
        if nranks > 1:
            if nccl_id is None:
                raise ValueError("a sharded system needs the NCCL unique id of rank 0")
            buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            self.ctx.call("hs_comm_init", buf)
        modes = {"subdomain": 0, "shared": 1, "kinds": 2}
        if maps not in modes:
            raise ValueError(f"maps must be 'subdomain', 'shared' or 'kinds', got {maps!r}")
        self.maps = maps
        self.ctx.call("hs_set_map_mode", modes[maps])
        # one-RHS BSP applies as a single dataflow launch: fused=True runs the
        # map-once plan (each map row read ~once per apply; equal to the step
        # sequence to rounding); fused=False one launch per step, also in
        # map-once form; fused="steps" / "literal" the literal SPEC arithmetic
        # as one launch / per step (bitwise equal to each other); R
        # right-hand sides run the DMMA dataflow launch (k_zmma2_df) under
        # fused=True too; an int is the raw hs_set_fused mask (8: the shared
        # maps' fused DMMA launch as well)
        if isinstance(fused, str):
            if fused not in ("steps", "literal"):
                raise ValueError(f"fused must be a bool, an int mask, 'steps' or 'literal', got {fused!r}")
            mask = 5 if fused == "steps" else 4
        elif isinstance(fused, bool):
            mask = 3 if fused else 0
        else:
            mask = int(fused)
        self.ctx.call("hs_set_fused", mask)
        self.home, cells = scatterer_cells(spec, partition)
        if self.home is not None:
            c = native.i32(cells)
            self.ctx.call("hs_set_dirichlet", self.home.i1, self.home.i2, native.iptr(c), len(c))
        t0 = time.perf_counter()
        if device >= 0:
            self.ctx.call("hs_factor")
        # device = -1: a plan-only system (lattice tables, windows, schedules,
        # exchange plans; no factorisation, every apply raises) -- the host side
        # of the boundary, usable without a GPU
        self.setup_time = time.perf_counter() - t0
        self._operators = None
        self.sweep = SweepConfig()
        self.configure(sweep or SweepConfig())

    # ---- row-band ranks on separate GPUs
    def enable_peer_memory(self):
        """Run the fused apply (and GMRES's A M v) over every rank's buffers
        through CUDA IPC: each rank exports its region, the handles are
        all-gathered in rank order (torch.distributed, already initialised when
        nranks > 1), and every rank maps its peers' regions.  Tiles then write
        their output blocks and completion counters directly in the owner's
        HBM (NVLink), replacing the per-step NCCL exchange.  With nranks = 1
        the same path runs on one GPU (the protocol minus the peers)."""
        h = (C.c_uint8 * 64)()
        self.ctx.call("hs_peer_export", h)
        allh = gather_peer_handles(bytes(h), self.rank, self.nranks)
        buf = (C.c_uint8 * len(allh)).from_buffer_copy(allh)
        self.ctx.call("hs_peer_open", buf, self.nranks)

    # ---- resources
    def close(self):
        """Release the device memory of this system now (maps, factors, work buffers)."""
        self.ctx.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    # ---- reference attributes
    @property
    def operators(self):
        if self._operators is None:
            self._operators = {i: SubdomainInfo.build(self.spec, self.imp, self.partition, i)
                               for i in self.partition.subdomains}
        return self._operators

    def configure(self, sweep: SweepConfig):
        """Windows and seam/residual options of the preconditioner."""
        P = self.partition
        for k, kind in ((0, "lower"), (1, "upper")):
            w = window_ranges(P.n1, P.n2, kind, sweep.blocks)
            lo, hi = native.i32([a for a, _ in w]), native.i32([b for _, b in w])
            self.ctx.call("hs_set_windows", k, native.iptr(lo), native.iptr(hi), len(w))
        seam = native.HS_SEAM_LITERAL if sweep.bsp_seam == "literal" else native.HS_SEAM_DEDUP
        if sweep.bsp_seam not in ("dedup", "literal"):
            raise ValueError(f"bsp_seam must be 'dedup' or 'literal', got {sweep.bsp_seam!r}")
        self.ctx.call("hs_set_precond_options", seam, int(bool(sweep.bsp_intermediate_residual)))
        self.sweep = sweep

    @contextlib.contextmanager
    def using(self, sweep: SweepConfig):
        """Run a block under another SweepConfig and restore the previous one."""
        prev = self.sweep
        if sweep == prev:
            yield self
            return
        self.configure(sweep)
        try:
            yield self
        finally:
            self.configure(prev)

    def _call_io(self, fn, g, pre=(), post=()):
        v = _Vec(self.layout.check(g), self.layout.size)
        out, optr = v.empty()
        self.ctx.call(fn, *pre, C.c_void_p(v.ptr), C.c_void_p(optr), v.R, *post, v.mem)
        return v.wrap(out)

    # ---- interface_system.py:98-162
    def compute_liftings(self, directions=None):
        """Lifting traces of the scatterer subdomain -> b (discretization.py:315-332,
        interface_system.py:98-113).  `directions`: list of incident directions for
        several right-hand sides (config 4)."""
        return {"b": self.rhs(directions), "directions": directions}

    def assemble_rhs(self, liftings) -> np.ndarray:
        return np.array(liftings["b"], copy=True)

    def rhs(self, directions=None) -> np.ndarray:
        home, data = lifting_data(self.spec, self.partition, directions)
        R = data.shape[1]
        out = np.zeros((self.layout.size, R), dtype=np.complex128)
        if home is not None:
            d = np.ascontiguousarray(data, dtype=np.complex128)
            self.ctx.call("hs_lifting_rhs", C.c_void_p(d.ctypes.data), R, C.c_void_p(out.ctypes.data),
                          native.HS_MEM_HOST)
        return out[:, 0] if directions is None else out

    def precondition_batch(self, rs, kind: str = "bsp", out=None):
        """Apply the preconditioner to a batch of independent HOST vectors
        (numpy arrays or CPU torch tensors, all the same shape; pinned torch
        tensors copy at full PCIe rate), pipelined so that each vector's
        host<->device copies overlap a neighbour's apply (hs_precond_batch).
        `out`: optional list of preallocated outputs of the inputs' kind."""
        if kind not in _PC:
            raise ValueError(f"unknown preconditioner {kind!r}")
        vs = [_Vec(self.layout.check(r), self.layout.size) for r in rs]
        if any(not v.cpu for v in vs):
            raise ValueError("precondition_batch takes host vectors (use bsp_apply for device tensors)")
        if len({v.shape for v in vs}) > 1:
            raise ValueError("precondition_batch: all vectors must have the same shape")
        if out is None:
            outs = [v.empty()[0] for v in vs]
        else:
            outs = list(out)
            if len(outs) != len(vs):
                raise ValueError("precondition_batch: one output per input")
        optrs = [(o.data_ptr() if hasattr(o, "data_ptr") else o.ctypes.data) for o in outs]
        n = len(vs)
        rp = (C.c_void_p * max(n, 1))(*[v.ptr for v in vs])
        zp = (C.c_void_p * max(n, 1))(*optrs)
        if n:
            self.ctx.call("hs_precond_batch", _PC[kind], rp, zp, n, vs[0].R)
        return outs if out is not None else [v.wrap(o) for v, o in zip(vs, outs)]

    def apply_scattering(self, g):
        return self._call_io("hs_apply", g, pre=(native.HS_APPLY_S,))

    def apply_interface_operator(self, g):
        return self._call_io("hs_apply", g, pre=(native.HS_APPLY_IMS,))

    def restricted_apply(self, g, source_groups, target_groups):
        src, tgt = native.i32(sorted(set(source_groups))), native.i32(sorted(set(target_groups)))
        v = _Vec(self.layout.check(g), self.layout.size)
        out, optr = v.empty()
        self.ctx.call("hs_restricted_apply", C.c_void_p(v.ptr), C.c_void_p(optr), v.R,
                      native.iptr(src), len(src), native.iptr(tgt), len(tgt), v.mem)
        return v.wrap(out)

    def materialize_dense(self) -> np.ndarray:
        size = self.layout.size
        if size > DENSE_GUARD:
            raise ValueError(f"dense guard exceeded: {size} > {DENSE_GUARD}")
        out = np.zeros((size, size), dtype=complex)
        for c0 in range(0, size, 512):
            c1 = min(size, c0 + 512)
            R = 1 << (c1 - c0 - 1).bit_length()
            E = np.zeros((size, R), dtype=complex)
            E[np.arange(c0, c1), np.arange(c1 - c0)] = 1.0
            out[:, c0:c1] = self.apply_scattering(E)[:, :c1 - c0]
        return out

    def reconstruct_solution(self, g, with_lifting: bool = True) -> np.ndarray:
        """Stitched global field u_i = v_i + w_i as an
        (N2 n) x (N1 n) complex array, y slow, computed on the GPU from the
        stored block factors (v_i: solve_local with the incoming traces of g,
        discretization.py:264-293; w_i: the lifting, :315-332)."""
        g = np.ascontiguousarray(np.asarray(self.layout.check(g)), dtype=np.complex128)
        if g.ndim != 1:
            raise ValueError("reconstruct_solution takes one right-hand side")
        n, P = self.n, self.partition
        field = np.zeros((P.n2 * n, P.n1 * n), dtype=np.complex128)
        lift = None
        if with_lifting:
            home, data = lifting_data(self.spec, P)
            if home is not None:
                lift = np.ascontiguousarray(data[:, 0])
        self.ctx.call("hs_reconstruct", C.c_void_p(g.ctypes.data),
                      C.c_void_p(lift.ctypes.data) if lift is not None else None,
                      C.c_void_p(field.ctypes.data), native.HS_MEM_HOST)
        return field

    def schur_map(self, i) -> np.ndarray:
        """Compact (k n) x (k n) map of subdomain i (faces W,S,N,E)."""
        i = MultiIndex(*i)
        k = len(self.partition.neighbors[i])
        K = k * self.n
        T = np.zeros((K, K), dtype=np.complex128)
        self.ctx.call("hs_get_schur", i.i1, i.i2, C.c_void_p(T.ctypes.data))
        return T

    # ---- SPEC.md:306-348
    def precondition(self, r, kind: str | None = None):
        kind = self.sweep.kind if kind is None else kind
        return self._call_io("hs_precond", r, pre=(_PC[kind],))

    def bsp_apply(self, b):
        return self.precondition(b, "bsp")

    def sgs_apply(self, r):
        return self.precondition(r, "sp")

    def bj_half_apply(self, r, direction: str):
        d = {"forward": 0, "backward": 1}[direction]
        return self._call_io("hs_half_apply", r, pre=(d,))

    def _single_window(self):
        ng = self.partition.n_groups
        one = native.i32([2]), native.i32([ng + 1])
        for k in (0, 1):
            self.ctx.call("hs_set_windows", k, native.iptr(one[0]), native.iptr(one[1]), 1 if ng >= 2 else 0)

    def forward_sweep(self, r):
        self._single_window()
        try:
            return self.bj_half_apply(r, "forward")
        finally:
            self.configure(self.sweep)

    def backward_sweep(self, r):
        self._single_window()
        try:
            return self.bj_half_apply(r, "backward")
        finally:
            self.configure(self.sweep)

    def step_schedule(self, kind: str | None = None):
        """[(step, phase, [MultiIndex])]."""
        kind = self.sweep.kind if kind is None else kind
        return schedule_records(self.ctx, self.partition, kind, self.sweep)

    # ---- SPEC.md:399-407 on the device
    def gmres(self, b, kind: str | None = None, tol: float = 1e-6, maxit: int = 200,
              arnoldi: str = "auto") -> GmresResult:
        """arnoldi = "auto" (one right-hand side: "cgs2g", on one GPU and
        across row bands; several, up to 128, on one GPU: "cgs2g" column by
        column; otherwise the MGS kernels -- a cluster kernel for small
        vectors, grid-wide otherwise, host-driven MGS with a reduction per
        inner product across bands), "mgs" (the MGS kernels for one
        right-hand side too: the SPEC's literal Arnoldi; k_mgs1c / k_mgs1 with
        M steps per grid barrier), "hostloop" (force the sharded MGS on one
        GPU or across bands), "grid" (force the generic grid-wide cooperative
        kernel k_mgs + k_givens), "cgs2" (classical
        Gram-Schmidt with one reorthogonalisation, iterations within +-1 of
        MGS) or "cgs2g" (CGS2 with the reorthogonalisation done on the
        coefficients through the device-kept Gram matrix: ONE reduction per
        iteration, the row-band default)."""
        kind = self.sweep.kind if kind is None else kind
        modes = {"auto": 0, "hostloop": 1, "grid": 2, "cgs2": 3, "cgs2g": 4, "mgs": 5}
        if arnoldi not in modes:
            raise ValueError(f"arnoldi must be one of {sorted(modes)}, got {arnoldi!r}")
        self.ctx.call("hs_set_gmres_mode", modes[arnoldi])
        v = _Vec(self.layout.check(b), self.layout.size)
        out, optr = v.empty()
        R = v.R
        self._last_R = R
        iters = np.zeros(R, dtype=np.int32)
        conv = np.zeros(R, dtype=np.int32)
        hist = np.zeros((maxit + 1, R), dtype=np.float64)
        t0 = time.perf_counter()
        self.ctx.call("hs_gmres", _PC[kind], C.c_void_p(v.ptr), C.c_void_p(optr), R, float(tol), int(maxit),
                      native.iptr(iters), hist.ctypes.data_as(C.POINTER(C.c_double)), native.iptr(conv), v.mem)
        wall = time.perf_counter() - t0
        if R == 1:
            h = list(hist[:iters[0] + 1, 0]) if iters[0] > 0 else []
            return GmresResult(v.wrap(out), h, int(iters[0]), bool(conv[0]), wall)
        return GmresResult(v.wrap(out), [list(hist[:iters[r] + 1, r]) for r in range(R)], iters.tolist(),
                           conv.astype(bool).tolist(), wall)


    def gmres_basis(self, ncols: int | None = None) -> np.ndarray:
        """The Arnoldi basis of the last gmres call, (L, ncols) complex128 for one
        right-hand side ((L, R, ncols) for R): SPEC.md:412's orthonormality
        invariant is checked on it (tests)."""
        avail = C.c_int(0)
        self.ctx.call("hs_gmres_basis", None, 0, C.byref(avail))
        ncols = avail.value if ncols is None else int(ncols)
        L = self.layout.size
        out = np.empty(ncols * self._last_R * L, dtype=np.complex128)
        self.ctx.call("hs_gmres_basis", C.c_void_p(out.ctypes.data), ncols, C.byref(avail))
        V = out.reshape(ncols, L, self._last_R)
        return V[:, :, 0].T.copy() if self._last_R == 1 else np.moveaxis(V, 0, -1).copy()


InterfaceSystem = GpuInterfaceSystem


def schedule_records(ctx, partition, kind, sweep):
    recs = []
    subs = partition.subdomains
    raw = ctx.schedule(_PC[kind])
    phases = {0: "forward", 1: "residual", 2: "backward"}
    cur = None
    for step, ph, s in raw:
        if cur is None or cur[0] != step:
            cur = (int(step), phases[int(ph)], [])
            recs.append(cur)
        cur[2].append(subs[int(s)])
    if kind == "bsp" and sweep.bsp_intermediate_residual and sweep.count_residual_steps:
        nf = sum(1 for r in recs if r[1] == "forward")
        res = (nf + 1, "residual", list(subs))
        recs = recs[:nf] + [res] + [(t + 1, ph, ss) for t, ph, ss in recs[nf:]]
    return recs
