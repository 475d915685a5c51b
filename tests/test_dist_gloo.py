"""CPU, multi-process (gloo): the row-band sharded BSP / (I - S) applies.

Each rank owns a band of subdomain rows, applies only its
subdomains' Schur maps (oracle, test infrastructure) and exchanges the outputs
that cross a band edge with its neighbours using the native exchange plan
(hs_exchange_plan: the same slot order the NCCL send/recv path of libhsb200
uses), applying the epilogue on receipt exactly like k_recv_epi.  The owned
blocks must equal the single-process result.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import oracle_problem
from paper_2209_10886_b200.configs import small_case

CASE = small_case(4, 6, 8)
CASE5 = dict(small_case(5, 7, 8), center=(2.5, 5.0), radius=0.9)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class Band:
    def __init__(self, case, rank, world, blocks):
        from oracle import Interface
        from oracle.lattice import windows
        from paper_2209_10886_b200 import native
        from paper_2209_10886_b200.indexing import window_ranges
        self.prob, self.lat = oracle_problem(case)
        self.itf = Interface(self.prob, self.lat, backend="schur")
        self.n = self.prob.n
        self.rank, self.world = rank, world
        self.ctx = native.Context(-1, case["n1"], case["n2"], self.n, 0.1, 1.0, 1j, rank=rank, nranks=world)
        for k, kd in ((0, "lower"), (1, "upper")):
            w = window_ranges(case["n1"], case["n2"], kd, blocks)
            lo, hi = native.i32([a for a, _ in w]), native.i32([b for _, b in w])
            self.ctx.call("hs_set_windows", k, native.iptr(lo), native.iptr(hi), len(w))
        self.lower = windows(case["n1"], case["n2"], "lower", blocks)
        self.upper = windows(case["n1"], case["n2"], "upper", blocks)
        self.owner = self.ctx.block_owner()
        self.sub_rank = {s: int(self.owner[self.lat.first_block[s] - 1]) for s in self.lat.subs}

    def blk(self, m):
        return slice(m * self.n, (m + 1) * self.n)

    def outputs(self, s, src, faces):
        """(target block, y) for the given compact faces of subdomain s."""
        T = self.itf.T[s]
        x = src[self.itf.in_slice(s)]
        out = []
        for q in faces:
            f, j = self.lat.faces[s][q]
            y = T[q * self.n:(q + 1) * self.n] @ x
            out.append((self.lat.m_index(j, s) - 1, y))
        return out

    def exchange(self, kind, t, remote, apply):
        """Send raw outputs in plan slot order, receive, apply epilogue."""
        reqs, recvs = [], []
        for peer in (self.rank - 1, self.rank + 1):
            if not 0 <= peer < self.world:
                continue
            plan = self.ctx.exchange_plan(kind, peer)
            plan = plan[plan[:, 0] == t] if len(plan) else plan
            if len(plan):
                buf = np.zeros((len(plan), self.n), dtype=complex)
                for _, b, slot in plan:
                    buf[slot] = remote[int(b)]
                reqs.append(dist.isend(torch.view_as_real(torch.from_numpy(buf)).contiguous(), peer))
            rplan = self.ctx.exchange_plan(kind, peer, recv=True)
            rplan = rplan[rplan[:, 0] == t] if len(rplan) else rplan
            if len(rplan):
                rb = torch.zeros((len(rplan), self.n, 2), dtype=torch.float64)
                reqs.append(dist.irecv(rb, peer))
                recvs.append((rplan, rb))
        for r in reqs:
            r.wait()
        for rplan, rb in recvs:
            vals = torch.view_as_complex(rb).numpy()
            for _, b, slot in rplan:
                apply(int(b), vals[slot])

    def run_step(self, kind, t, items, apply):
        remote = {}
        for s, src, faces in items:
            if self.sub_rank[s] != self.rank:
                continue
            for b, y in self.outputs(s, src, faces):
                if self.owner[b] == self.rank:
                    apply(b, y)
                else:
                    remote[b] = y
        self.exchange(kind, t, remote, apply)

    def half_items(self, direction, t, state, inp):
        wins = self.lower if direction == 0 else self.upper
        items = []
        for lo, hi in wins:
            if t > hi - lo:
                continue
            g = lo + t - 1 if direction == 0 else hi - t + 1
            src = inp if t == 1 else state
            for s in self.lat.groups.get(g, []):
                nl = sum(1 for f, _ in self.lat.faces[s] if f in (0, 1))
                k = len(self.lat.faces[s])
                faces = range(nl, k) if direction == 0 else range(0, nl)
                if len(faces):
                    items.append((s, src, faces))
        return items

    def bsp(self, b):
        zl = b.copy()
        depth = max(hi - lo for lo, hi in self.lower)
        for t in range(1, depth + 1):
            def acc(blk, y):
                zl[self.blk(blk)] += y
            self.run_step(0, t - 1, self.half_items(0, t, zl, b), acc)
        rp, w, z = np.zeros_like(b), np.zeros_like(b), np.zeros_like(b)

        def resid(blk, y):
            sl = self.blk(blk)
            v = b[sl] - (zl[sl] - y)
            rp[sl], w[sl], z[sl] = v, v, zl[sl] + v
        full = [(s, zl, range(len(self.lat.faces[s]))) for s in self.lat.subs]
        self.run_step(2, 0, full, resid)
        depth = max(hi - lo for lo, hi in self.upper)
        for t in range(1, depth + 1):
            def acc2(blk, y):
                w[self.blk(blk)] += y
                z[self.blk(blk)] += y
            self.run_step(1, t - 1, self.half_items(1, t, w, rp), acc2)
        return z

    def map_once(self, which):
        import ctypes as C
        cnt = C.c_int(0)
        self.ctx.call("hs_map_once_plan", which, None, 0, C.byref(cnt))
        buf = (C.c_int32 * max(cnt.value, 1))()
        self.ctx.call("hs_map_once_plan", which, buf, cnt.value, C.byref(cnt))
        return np.frombuffer(buf, dtype=np.int32)[:cnt.value]

    def mo_items(self, which, src):
        v = self.map_once(which).reshape(-1, 4)
        return [((int(i1), int(i2)), src, range(int(lo) // self.n, int(hi) // self.n)) for i1, i2, lo, hi in v]

    def bsp_map_once(self, b):
        """The per-step map-once BSP of the library's row-band path: forward
        half, W/S blocks of exact forward writers filled (r' = 0), the residual
        step on the map-once rows (kind 3), backward half."""
        zl = b.copy()
        depth = max(hi - lo for lo, hi in self.lower)
        for t in range(1, depth + 1):
            def acc(blk, y):
                zl[self.blk(blk)] += y
            self.run_step(0, t - 1, self.half_items(0, t, zl, b), acc)
        rp, w, z = np.zeros_like(b), np.zeros_like(b), np.zeros_like(b)
        for blk in self.map_once(3):
            sl = self.blk(int(blk))
            rp[sl] = w[sl] = 0
            z[sl] = zl[sl]

        def resid(blk, y):
            sl = self.blk(blk)
            v = b[sl] - (zl[sl] - y)
            rp[sl], w[sl], z[sl] = v, v, zl[sl] + v
        self.run_step(3, 0, self.mo_items(0, zl), resid)
        depth = max(hi - lo for lo, hi in self.upper)
        for t in range(1, depth + 1):
            def acc2(blk, y):
                w[self.blk(blk)] += y
                z[self.blk(blk)] += y
            self.run_step(1, t - 1, self.half_items(1, t, w, rp), acc2)
        return z, rp, w

    def ims_map_once(self, r, rp, w):
        """(I - S) z right after bsp_map_once(r): r on the N/E blocks of final
        backward writers, r - T_up w (kind 4), (r - rp) + (w - T_low w) on the
        window starts' lower rows (kind 5)."""
        out = np.zeros_like(r)
        for blk in self.map_once(4):
            sl = self.blk(int(blk))
            out[sl] = r[sl]

        def ims(blk, y):
            sl = self.blk(blk)
            out[sl] = r[sl] - y

        def late(blk, y):
            sl = self.blk(blk)
            out[sl] = (r[sl] - rp[sl]) + (w[sl] - y)
        self.run_step(4, 0, self.mo_items(1, w), ims)
        self.run_step(5, 0, self.mo_items(2, w), late)
        return out

    def apply_A(self, g):
        out = np.zeros_like(g)

        def ims(blk, y):
            out[self.blk(blk)] = g[self.blk(blk)] - y
        full = [(s, g, range(len(self.lat.faces[s]))) for s in self.lat.subs]
        self.run_step(2, 0, full, ims)
        return out

    def owned_mask(self):
        return np.repeat(self.owner == self.rank, self.n)

    def gmres(self, b, tol=1e-6, maxit=200):
        """Right-preconditioned MGS GMRES with every inner product reduced over
        the ranks (the algorithm of gmres_arnoldi_dist: partial dots over owned
        blocks, one all-reduce each, Givens replicated on every rank)."""
        from oracle.gmres import givens
        m = self.owned_mask()

        def dot(u, v):
            t = torch.tensor([complex(np.vdot(u[m], v[m]))], dtype=torch.complex128)
            t = torch.view_as_real(t).contiguous()
            dist.all_reduce(t)
            return complex(t[0, 0].item(), t[0, 1].item())

        beta = abs(dot(b, b)) ** 0.5
        V = [np.where(m, b / beta, 0)]
        H = np.zeros((maxit + 1, maxit), complex)
        cs, sn = np.zeros(maxit), np.zeros(maxit, complex)
        g = np.zeros(maxit + 1, complex)
        g[0] = beta
        k_done = 0
        for k in range(maxit):
            w = self.apply_A(self.bsp(V[k]))
            w = np.where(m, w, 0)
            for j in range(k + 1):
                H[j, k] = dot(V[j], w)
                w = w - H[j, k] * V[j]
            hn = abs(dot(w, w)) ** 0.5
            H[k + 1, k] = hn
            for j in range(k):
                t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
                H[j + 1, k] = -np.conj(sn[j]) * H[j, k] + cs[j] * H[j + 1, k]
                H[j, k] = t
            c, s_ = givens(H[k, k], H[k + 1, k].real)
            cs[k], sn[k] = c, s_
            H[k, k] = c * H[k, k] + s_ * H[k + 1, k]
            H[k + 1, k] = 0
            g[k + 1] = -np.conj(s_) * g[k]
            g[k] = c * g[k]
            k_done = k + 1
            if abs(g[k + 1]) / beta <= tol:
                break
            V.append(w / hn)
        y = np.linalg.solve(np.triu(H[:k_done, :k_done]), g[:k_done])
        u = sum(y[i] * V[i] for i in range(k_done))
        return self.bsp(u), k_done


    def gmres_cgs2g(self, b, tol=1e-6, maxit=200):
        """The row-band default Arnoldi (gmres_arnoldi_cgsg): CGS2 with the
        reorthogonalisation done on the coefficients through the Gram matrix
        G = V^H V -- ONE all-reduce per iteration of [V^H w, V^H v_k, ||w||^2]
        over the owned blocks; c = 2h - G h, w'' = w - V c, ||w''||^2 =
        ||w||^2 - 2 Re(c^H h) + c^H G c.  Returns (x, iterations, all-reduces)."""
        from oracle.gmres import givens
        m = self.owned_mask()
        nred = [0]

        def allreduce(vec):
            t = torch.view_as_real(torch.tensor(np.asarray(vec, complex))).contiguous()
            dist.all_reduce(t)
            nred[0] += 1
            return t[:, 0].numpy() + 1j * t[:, 1].numpy()

        beta = abs(allreduce([np.vdot(b[m], b[m])])[0]) ** 0.5
        V = [np.where(m, b / beta, 0)]
        Gm = np.zeros((maxit + 1, maxit + 1), complex)
        H = np.zeros((maxit + 1, maxit), complex)
        cs, sn = np.zeros(maxit), np.zeros(maxit, complex)
        g = np.zeros(maxit + 1, complex)
        g[0] = beta
        k_done = 0
        for k in range(maxit):
            w = np.where(m, self.apply_A(self.bsp(V[k])), 0)
            loc = [np.vdot(V[j][m], w[m]) for j in range(k + 1)] + \
                  [np.vdot(V[j][m], V[k][m]) for j in range(k + 1)] + [np.vdot(w[m], w[m])]
            red = allreduce(loc)
            h, gk, w2 = red[:k + 1], red[k + 1:2 * k + 2], red[-1].real
            Gm[k, :k + 1] = gk                       # <v_j, v_k>
            L = np.tril(Gm[:k + 1, :k + 1])          # L[i][j] = v_j^H v_i, j <= i
            Gfull = np.conj(L) + np.tril(L, -1).T    # G[i][j] = v_i^H v_j
            c = 2 * h - Gfull @ h
            q = w2 - 2 * np.real(np.vdot(c, h)) + np.real(np.vdot(c, Gfull @ c))
            hn = max(q, 0.0) ** 0.5
            w = w - sum(c[j] * V[j] for j in range(k + 1))
            H[:k + 1, k] = c
            H[k + 1, k] = hn
            for j in range(k):
                t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
                H[j + 1, k] = -np.conj(sn[j]) * H[j, k] + cs[j] * H[j + 1, k]
                H[j, k] = t
            c_, s_ = givens(H[k, k], H[k + 1, k].real)
            cs[k], sn[k] = c_, s_
            H[k, k] = c_ * H[k, k] + s_ * H[k + 1, k]
            H[k + 1, k] = 0
            g[k + 1] = -np.conj(s_) * g[k]
            g[k] = c_ * g[k]
            k_done = k + 1
            if abs(g[k + 1]) / beta <= tol:
                break
            V.append(w / hn)
        y = np.linalg.solve(np.triu(H[:k_done, :k_done]), g[:k_done])
        u = sum(y[i] * V[i] for i in range(k_done))
        return self.bsp(u), k_done, nred[0]


def _worker(rank, world, port, case, blocks, q, with_gmres=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Interface, Preconditioner
        band = Band(case, rank, world, blocks)
        rng = np.random.default_rng(7)
        r = rng.standard_normal(band.itf.size) + 1j * rng.standard_normal(band.itf.size)
        z = band.bsp(r)
        a = band.apply_A(r)
        ref_itf = Interface(band.prob, band.lat, backend="schur")
        zr = Preconditioner(ref_itf, "bsp", blocks=blocks)(r)
        ar = ref_itf.apply_A(r)
        m = band.owned_mask()
        res = [rank, float(np.abs(z[m] - zr[m]).max() / np.abs(zr).max()),
               float(np.abs(a[m] - ar[m]).max() / np.abs(ar).max()), int(m.sum())]
        if with_gmres:
            from oracle.gmres import gmres
            from oracle.schur import lifting_traces
            home, tr = lifting_traces(band.prob, band.lat)
            b = np.zeros(ref_itf.size, complex)
            for f, j in band.lat.faces[home]:
                b[ref_itf.block(band.lat.m_index(j, home))] = tr[f]
            x, its = band.gmres(b)
            ref = gmres(ref_itf.apply_A, Preconditioner(ref_itf, "bsp", blocks=blocks), b, tol=1e-6, maxit=200)
            res += [its, ref.iterations, float(np.abs(x[m] - ref.x[m]).max() / np.abs(ref.x).max())]
            xg, itg, nred = band.gmres_cgs2g(b)
            res += [itg, nred, float(np.abs(xg[m] - ref.x[m]).max() / np.abs(ref.x).max())]
        q.put(tuple(res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world,blocks", [(CASE, 2, None), (CASE, 3, 2), (CASE5, 2, 4), (CASE5, 3, None)])
def test_sharded_bsp_matches_single_process(case, world, blocks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, blocks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    L = None
    total = 0
    for rank, ez, ea, owned in [r[:4] for r in res]:
        assert ez < 1e-13, (rank, ez)
        assert ea < 1e-13, (rank, ea)
        total += owned
    from oracle.lattice import Lattice
    assert total == Lattice(case["n1"], case["n2"]).n_pairs * case["n"]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gmres_matches_single_process(world):
    """Row-band GMRES (inner products all-reduced over the ranks, as in
    gmres_arnoldi_dist) converges in the same iterations to the same x."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASE5, None, q, True)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in res:
        its, ref_its, ex = r[4], r[5], r[6]
        assert its == ref_its, (its, ref_its)
        assert ex < 1e-10, ex
        # the row-band default (CGS2, Gram-corrected): one all-reduce per
        # iteration (+ the initial norm), the same iterations and x
        itg, nred, exg = r[7], r[8], r[9]
        assert itg == ref_its, (itg, ref_its)
        assert nred == itg + 1, (nred, itg)
        assert exg < 1e-10, exg


# ---- the multi-GPU peer-memory protocol, emulated by processes -------------
# Each process is one row-band rank running the tiles hs_fused_plan lists for
# it (the global ticket order of the map-once plan, filtered to its
# subdomains), reading and writing the vectors and completion counters of
# every block in its OWNER's region -- shared memory standing in for the
# peers' HBM mapped through CUDA IPC.  A tile waits on the owners' counters,
# computes its 32-row strip product (oracle maps), finishes the rows with the
# kernel's epilogue in the owner's vectors and bumps the owners' counters.
# Every counter has one writer (the rank of the block's writer subdomain), so
# plain stores suffice; x86 keeps stores and loads in order.
FV_R, FV_ZL, FV_RP, FV_W, FV_Z, FV_WOUT = range(6)


def _parse_plan(v):
    out, i = [], 0
    while i < len(v):
        rec = [int(x) for x in v[i:i + 12]]
        nd = rec[11]
        deps = [(int(v[i + 12 + 2 * d]), int(v[i + 13 + 2 * d])) for d in range(nd)]
        out.append((rec, deps))
        i += 12 + 2 * nd
    return out


def _tile_signals(band, rec):
    """Blocks a tile completes (the kernel's tile_signal rule)."""
    i1, i2, rlo, rhi, c0, c1, alt, row0, phase, flags, rmask, _ = rec
    s, n = (i1, i2), band.n
    if phase in (3, 5):
        return []
    nlow = sum(1 for f, _ in band.lat.faces[s] if f in (0, 1))
    r0, r1 = max(rlo, row0), min(rhi, row0 + 32)
    return [band.lat.m_index(band.lat.faces[s][f][1], s) - 1 for f in range(r0 // n, (r1 - 1) // n + 1)
            if phase <= 1 or f < nlow]


def _tile_wout(band, rec):
    """Blocks whose wout rows a tile writes (counted for the owner's drain)."""
    i1, i2, rlo, rhi, c0, c1, alt, row0, phase, flags, rmask, _ = rec
    if not (phase in (3, 5) or (phase in (2, 4) and flags & 2)):
        return []
    s, n = (i1, i2), band.n
    r0, r1 = max(rlo, row0), min(rhi, row0 + 32)
    return [band.lat.m_index(band.lat.faces[s][f][1], s) - 1 for f in range(r0 // n, (r1 - 1) // n + 1)]


def _run_peer_tiles(band, plan, V, CNT, base=None, WCNT=None):
    """base: per-block completion count at the start of this apply (epoch
    protocol: counters are never reset), else zero."""
    import time
    n = band.n
    for rec, deps in plan:
        i1, i2, rlo, rhi, c0, c1, alt, row0, phase, flags, rmask, _ = rec
        s = (i1, i2)
        for b, cnt in deps:
            o = band.owner[b]
            want = cnt + (0 if base is None else base[b])
            while CNT[o, b] < want:
                time.sleep(0)
        me = band.rank
        k = len(band.lat.faces[s])
        K = k * n
        nlow = sum(1 for f, _ in band.lat.faces[s] if f in (0, 1))
        sl = band.itf.in_slice(s)
        x1v = {0: FV_R if alt else FV_ZL, 1: FV_ZL, 2: FV_RP if alt else FV_W, 3: FV_Z, 4: FV_ZL}.get(phase, FV_W)
        xs = V[me, x1v, sl].copy()
        r_in = V[me, FV_R, sl]
        for q in range(k):
            if (rmask >> q) & 1:
                xs[q * n:(q + 1) * n] = r_in[q * n:(q + 1) * n]
        if flags & 4:  # FT_DIFF
            xs = xs - (r_in if phase == 1 else V[me, FV_RP, sl])
        cols = np.arange(K)
        xs[(cols < c0) | (cols >= c1)] = 0
        r0, r1 = max(rlo, row0), min(rhi, row0 + 32)
        T = band.itf.T[s]
        y1 = T[r0:r1] @ xs
        y2 = T[r0:r1] @ V[me, FV_RP if alt else FV_W, sl] if phase == 4 else None
        for row in range(r0, r1):
            f, p = divmod(row, n)
            _, j = band.lat.faces[s][f]
            blk = band.lat.m_index(j, s) - 1
            o = band.owner[blk]
            t = blk * n + p
            low, zr = f < nlow, (rmask >> (4 + f)) & 1
            Vo = V[o]
            zb = Vo[FV_R, t] if zr else Vo[FV_ZL, t]
            a = y1[row - r0]
            if phase == 0:
                Vo[FV_ZL, t] = zb + a
                if flags & 1:  # FT_ZERO
                    Vo[FV_RP, t] = Vo[FV_W, t] = 0
                    Vo[FV_Z, t] = zb + a
            elif phase == 1:
                v = a if flags & 4 else Vo[FV_R, t] - (zb - a)
                Vo[FV_RP, t] = Vo[FV_W, t] = v
                Vo[FV_Z, t] = zb + v
            elif phase == 2:
                if low:
                    Vo[FV_W, t] += a
                    Vo[FV_Z, t] += a
                    if flags & 2:
                        Vo[FV_WOUT, t] = Vo[FV_R, t]
                else:
                    Vo[FV_WOUT, t] = Vo[FV_R, t] - a
            elif phase == 4:
                b2 = y2[row - r0]
                if low:
                    v = Vo[FV_R, t] - (zb - a)
                    Vo[FV_RP, t] = v
                    Vo[FV_W, t] = v + b2
                    Vo[FV_Z, t] = (zb + v) + b2
                    if flags & 2:
                        Vo[FV_WOUT, t] = Vo[FV_R, t]
                else:
                    Vo[FV_WOUT, t] = Vo[FV_R, t] - b2
            elif phase == 5:
                if low and not flags & 4:
                    Vo[FV_WOUT, t] = (Vo[FV_R, t] - Vo[FV_RP, t]) + (Vo[FV_W, t] - a)
                else:
                    Vo[FV_WOUT, t] = Vo[FV_R, t] - a
        for blk in _tile_signals(band, rec):
            CNT[band.owner[blk], blk] += 1
        if WCNT is not None:
            for blk in _tile_wout(band, rec):
                WCNT[band.owner[blk], blk] += 1


def _plan_of(band, ims, rank):
    import ctypes as C
    cnt = C.c_int(0)
    band.ctx.call("hs_fused_plan", int(ims), rank, None, 0, C.byref(cnt))
    buf = (C.c_int32 * cnt.value)()
    band.ctx.call("hs_fused_plan", int(ims), rank, buf, cnt.value, C.byref(cnt))
    return _parse_plan(np.frombuffer(buf, dtype=np.int32))


def _peer_epoch_worker(rank, world, port, case, blocks, vbuf, cbuf, fbuf, napply, q, wbuf=None):
    """The barrier-free epoch protocol of the GPU path: for apply e every rank
    copies in its r, posts e, waits for every rank's post, runs its tiles with
    dependency counts offset by the blocks' totals of the previous applies,
    drains its own blocks (counter = e * total) and reads its z -- no barrier
    between applies; BSP and A M v applies alternate."""
    import time
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        band = Band(case, rank, world, blocks)
        plans = {ims: _plan_of(band, ims, rank) for ims in (False, True)}
        wt = {}
        for ims in (False, True):  # signals per block per apply: every rank's tiles
            w = np.zeros(len(band.owner), dtype=np.int64)
            for r in range(world):
                for rec, _ in _plan_of(band, ims, r):
                    for b in _tile_signals(band, rec):
                        w[b] += 1
            wt[ims] = w
        assert np.array_equal(wt[False], wt[True])  # one total per block for both plans
        W = wt[False]
        WW = np.zeros(len(band.owner), dtype=np.int64)  # wout writes per block per A M v apply
        for r in range(world):
            for rec, _ in _plan_of(band, True, r):
                for b in _tile_wout(band, rec):
                    WW[b] += 1
        V = vbuf.numpy().view(complex)[..., 0]
        CNT, FLAG = cbuf.numpy(), fbuf.numpy()
        WCNT = wbuf.numpy()
        n_ims = 0
        own = np.where(band.owner == rank)[0]
        m = band.owned_mask()
        from oracle import Preconditioner
        pc = Preconditioner(band.itf, "bsp", blocks=blocks)
        dist.barrier()  # buffers zeroed by the parent, every process started
        errs = []
        for e in range(1, napply + 1):
            ims = e % 2 == 0
            rng = np.random.default_rng(100 + e)
            r = rng.standard_normal(V.shape[2]) + 1j * rng.standard_normal(V.shape[2])
            V[rank, FV_R] = r
            FLAG[rank] = e  # post this epoch's inputs
            for g in range(world):
                while FLAG[g] < e:
                    time.sleep(0)
            n_ims += int(ims)
            _run_peer_tiles(band, plans[ims], V, CNT, base=(e - 1) * W, WCNT=WCNT)
            for b in own:  # drain: every write into this rank's blocks has landed
                while CNT[rank, b] < e * W[b]:
                    time.sleep(0)
                while ims and WCNT[rank, b] < n_ims * WW[b]:  # and the wout rows (A M v)
                    time.sleep(0)
            ref = pc.bsp_apply(r)
            got = V[rank, FV_WOUT if ims else FV_Z].copy()
            want = band.itf.apply_A(ref) if ims else ref
            errs.append(float(np.abs(got[m] - want[m]).max() / np.abs(want).max()))
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


def _peer_worker(rank, world, port, case, blocks, vbuf, cbuf, ims, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C
        band = Band(case, rank, world, blocks)
        cnt = C.c_int(0)
        band.ctx.call("hs_fused_plan", int(ims), rank, None, 0, C.byref(cnt))
        buf = (C.c_int32 * cnt.value)()
        band.ctx.call("hs_fused_plan", int(ims), rank, buf, cnt.value, C.byref(cnt))
        plan = _parse_plan(np.frombuffer(buf, dtype=np.int32))
        V = vbuf.numpy().view(complex)[..., 0]  # [world, 6, L]
        CNT = cbuf.numpy()
        rng = np.random.default_rng(3)
        r = rng.standard_normal(V.shape[2]) + 1j * rng.standard_normal(V.shape[2])
        V[rank, FV_R] = r
        CNT[rank] = 0
        dist.barrier()  # every rank's inputs in place, counters reset
        _run_peer_tiles(band, plan, V, CNT)
        dist.barrier()  # every write into this rank's blocks has landed
        from oracle import Preconditioner
        ref = Preconditioner(band.itf, "bsp", blocks=blocks).bsp_apply(r)
        m = band.owned_mask()
        ez = float(np.abs(V[rank, FV_Z][m] - ref[m]).max() / np.abs(ref).max())
        ew = 0.0
        if ims:
            refw = band.itf.apply_A(ref)
            ew = float(np.abs(V[rank, FV_WOUT][m] - refw[m]).max() / np.abs(refw).max())
        q.put((rank, len(plan), ez, ew))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world,blocks,ims", [(CASE, 2, None, False), (CASE, 3, 2, True),
                                                    (CASE5, 2, 4, True), (CASE5, 3, None, False)])
def test_peer_memory_protocol_matches_oracle(case, world, blocks, ims):
    """The fused apply over peer memory (hs_peer_open's path) with the ranks
    as processes and shared memory as the peers' HBM: BSP z (and GMRES's
    (I - S) z) on every rank's blocks equal the single-process oracle."""
    from oracle.lattice import Lattice
    L = Lattice(case["n1"], case["n2"]).n_pairs * case["n"]
    npairs = Lattice(case["n1"], case["n2"]).n_pairs
    vbuf = torch.zeros(world, 6, L, 2, dtype=torch.float64).share_memory_()
    cbuf = torch.zeros(world, npairs, dtype=torch.int64).share_memory_()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, case, blocks, vbuf, cbuf, ims, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(r[1] for r in res) > 0
    for rank, ntiles, ez, ew in res:
        assert ez < 1e-12, (rank, ez)
        assert ew < 1e-12, (rank, ew)


@pytest.mark.parametrize("case,world,blocks", [(CASE, 2, None), (CASE5, 3, 4)])
def test_peer_memory_epoch_protocol(case, world, blocks):
    """Four back-to-back applies (BSP, A M v, BSP, A M v) over the peer
    buffers with the epoch protocol and no barrier between them: every rank's
    blocks equal the oracle each time.  (The wout rows of the A M v plan are
    written by tiles that signal no completion; without their own counters
    and drain a rank read its (I - S) z before a peer's late tile had written
    it -- this test caught that race intermittently.)"""
    from oracle.lattice import Lattice
    lat = Lattice(case["n1"], case["n2"])
    L = lat.n_pairs * case["n"]
    vbuf = torch.zeros(world, 6, L, 2, dtype=torch.float64).share_memory_()
    cbuf = torch.zeros(world, lat.n_pairs, dtype=torch.int64).share_memory_()
    fbuf = torch.zeros(world, dtype=torch.int64).share_memory_()
    wbuf = torch.zeros(world, lat.n_pairs, dtype=torch.int64).share_memory_()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_epoch_worker, args=(r, world, port, case, blocks, vbuf, cbuf, fbuf, 4, q, wbuf))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errs in res:
        assert len(errs) == 4 and max(errs) < 1e-12, (rank, errs)


def _mo_worker(rank, world, port, case, blocks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        band = Band(case, rank, world, blocks)
        from oracle import Preconditioner
        rng = np.random.default_rng(11)
        r = rng.standard_normal(band.itf.size) + 1j * rng.standard_normal(band.itf.size)
        ref = Preconditioner(band.itf, "bsp", blocks=blocks).bsp_apply(r)
        z, rp, w = band.bsp_map_once(r)
        out = band.ims_map_once(r, rp, w)
        m = band.owned_mask()
        refw = band.itf.apply_A(ref)
        q.put((rank, float(np.abs(z[m] - ref[m]).max() / np.abs(ref).max()),
               float(np.abs(out[m] - refw[m]).max() / np.abs(refw).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world,blocks", [(CASE, 2, None), (CASE, 3, 2), (CASE5, 2, 4), (CASE5, 3, None)])
def test_sharded_map_once_per_step(case, world, blocks):
    """The row-band per-step path in map-once form (the NCCL-exchange fallback
    for R right-hand sides / no peer memory): the library's map-once tables
    and fill lists (hs_map_once_plan) and their band-crossing exchange plans
    (hs_exchange_plan kinds 3-5) give the oracle's BSP z and (I - S) z on
    every rank's blocks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mo_worker, args=(r, world, port, case, blocks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ez, ew in res:
        assert ez < 1e-13 and ew < 1e-13, (rank, ez, ew)


def _handles_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2209_10886_b200.interface_system import gather_peer_handles
        mine = bytes([rank + 1]) * 64
        allh = gather_peer_handles(mine, rank, world)
        try:
            gather_peer_handles(mine, rank, world + 1)
            bad = False
        except ValueError:
            bad = True
        q.put((rank, allh, bad))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_handle_exchange(world):
    """The host side of hs_peer_open: the ranks' 64-byte IPC handles are
    all-gathered in rank order (the layout hs_peer_open reads), and a rank /
    world mismatch with the process group is refused."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handles_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = b"".join(bytes([r + 1]) * 64 for r in range(world))
    for rank, allh, bad in res:
        assert allh == want and bad, rank
