#!/usr/bin/env python
"""Benchmark of the B200 hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

A *step* is one block-Jacobi sweeping-preconditioner (BSP) apply z = M r over
one synthetic interface vector (seeded complex normal) of the configured
problem -- by default BASELINE config 5 (32x16 subdomains of 256x256 cells,
8 blocks, 7.9 GB of Schur maps: far larger than the 126 MB L2, so no flush
is needed between steps).  `value` is applies/s of the whole job with the
vector resident in HBM (CUDA events on the library's stream, max over
ranks); `e2e` is the same through the C ABI with pinned host buffers
(host->device copy of r and device->host copy of z inside every step).
The line also reports the roofline of the dominant kernel (the batched
step-apply, timed per launch with CUDA events), GMRES time-to-solution, the
CPU baseline (the oracle port of the reference path on the host cores) and
the SM clocks seen during the timed region.

`--impl reference` times the reference algorithm on the host cores instead:
real BSP applies through the reference loop (oracle restatement, bitwise the
reference; SuperLU solves with the 2 distinct factors shared, every S
application's subdomain solves on all host cores via forked processes), each
step a bounded sample, plus the projected GMRES time-to-solution.  That arm
imports no product code.
Under torchrun with N > 1 the subdomain rows are sharded over the ranks
(strong scaling: the apply is split; traces cross band edges over NCCL).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GMRES time-to-solution; preconditioner applies/s and % of HBM roofline"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def problem(cfgno, blocks=None):
    from paper_2209_10886_b200.configs import CONFIGS, with_blocks
    from paper_2209_10886_b200.discretization import ProblemSpec, Scatterer
    from paper_2209_10886_b200.indexing import Partition
    c = CONFIGS[cfgno] if blocks is None else with_blocks(CONFIGS[cfgno], blocks)
    ang = c["angle"] if c["angle"] is not None else 0.0
    spec = ProblemSpec(kappa=c["kappa"], cells_per_side=c["n"], subdomain_side=c["side"],
                       scatterer=Scatterer(tuple(c["center"]), c["radius"]),
                       incident_direction=(float(np.cos(ang)), float(np.sin(ang))))
    return c, spec, Partition(c["n1"], c["n2"])


def config_json(c, world, exchange=None):
    out = {"workload": f"{c['name']}: BSP apply, {c['n1']}x{c['n2']} subdomains of {c['n']}x{c['n']} cells, "
                        f"{'reference' if c['blocks'] is None else c['blocks']} blocks, {c['nrhs']} RHS",
            "lattice": [c["n1"], c["n2"]], "cells_per_side": c["n"], "grid": [c["n1"] * c["n"], c["n2"] * c["n"]],
            "kappa": c["kappa"], "blocks": c["blocks"], "nrhs": c["nrhs"], "tol": c["tol"],
            "parallelism": f"rowbands{world}" if world > 1 else "single",
            "l2": (f"inputs larger than L2: Schur maps {schur_bytes(c) / 1e9:.2f} GB >> 126 MB L2, no flush"
                   if schur_bytes(c) > 4 * 126e6 else "L2 NOT flushed: maps fit in L2 (report as L2-resident)")}
    if world > 1:
        out["exchange"] = exchange
    return out


def schur_bytes(c):
    """Bytes of the per-subdomain maps: 16 n^2 sum_i k_i^2."""
    n1, n2, n = c["n1"], c["n2"], c["n"]
    tot = 0
    for a in range(1, n1 + 1):
        for b in range(1, n2 + 1):
            k = (a > 1) + (a < n1) + (b > 1) + (b < n2)
            tot += k * k
    return 16.0 * n * n * tot


# ---------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, dev):
        self.p = None
        self.dev = dev
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(dev), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU baseline / reference arm
def load_configs():
    """The BASELINE config table, loaded from its file WITHOUT importing the
    product package (configs.py is plain data; importing
    paper_2209_10886_b200.indexing would map libhsb200.so into the reference
    arm's process)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_hs_configs", os.path.join(ROOT, "paper_2209_10886_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def host_info():
    """CPU model and logical core count of the host (SURVEY.md §8d reporting)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count(),
            "note": "the reference's thread pool gives no speed-up (SURVEY.md §2a): the subdomain solves of "
                    "each S application run in forked processes, one BLAS thread each"}


def reference_iterations(cfgno, blocks=None):
    """GMRES iterations of the reference arithmetic on this config, from its golden
    run (tests/golden/cfg*.npz; config 4 = config 2's geometry, per angle; config
    2 with another block count: the gm_iters_p{p} keys of the sweep golden)."""
    name = {4: "cfg2"}.get(cfgno, f"cfg{cfgno}")
    p = os.path.join(ROOT, "tests", "golden", f"{name}.npz")
    if not os.path.exists(p):
        return None, None
    sfx = f"_p{blocks}" if blocks is not None else ""
    with np.load(p) as G:
        if f"gm_iters{sfx}" not in G.files:
            return None, None
        return int(G[f"gm_iters{sfx}"]), (float(G[f"gm_time{sfx}"]) if f"gm_time{sfx}" in G.files else None)


class ReferenceCPU:
    """The reference's arithmetic on the host cores: the oracle's SuperLU back
    end (bitwise the reference's _scatter_one, tests/test_oracle_golden.py) with
    its 2 distinct factors shared (discretization.py:224-229), the BSP apply of
    the SPEC restatement (oracle/sweeps.py) over the reference loop
    restricted_apply / apply_interface_operator (interface_system.py:135-162:
    gather, zero-skip, solve, outgoing traces, scatter), every subdomain solve
    of an S application spread over `workers` forked processes
    (oracle/parallel.py).  No product code is imported."""

    def __init__(self, cfgno, workers=None, blocks=None):
        from oracle import Interface, Lattice, Preconditioner, Problem
        from oracle.parallel import ParInterface
        cm = load_configs()
        c = cm.CONFIGS[cfgno] if blocks is None else cm.with_blocks(cm.CONFIGS[cfgno], blocks)
        self.c = c
        ang = c["angle"] if c["angle"] is not None else 0.0
        prob = Problem(kappa=c["kappa"], n=c["n"], side=c["side"], center=tuple(c["center"]), radius=c["radius"],
                       direction=(float(np.cos(ang)), float(np.sin(ang))))
        t0 = time.perf_counter()
        self.itf = Interface(prob, Lattice(c["n1"], c["n2"]), share_factors=True)
        self.setup_s = time.perf_counter() - t0
        self.P = ParInterface(self.itf, workers)
        self.workers = self.P.workers
        self.pc = Preconditioner(self.P, "bsp", blocks=c["blocks"])
        rng = np.random.default_rng(1234)
        self.r = rng.standard_normal(self.itf.size) + 1j * rng.standard_normal(self.itf.size)
        self.R = int(c["nrhs"])  # the reference has one right-hand side: R applies per multi-RHS apply
        self._stages = None
        self.solves_per_apply = None
        self.P.apply_A(self.r)  # warm: every worker has touched its share of the operators and factors

    def close(self):
        self.P.close()

    def time_apply(self):
        """One full BSP apply: (seconds, subdomain solves)."""
        s0, t0 = self.P.solves, time.perf_counter()
        self.pc.bsp_apply(self.r)
        dt, ns = time.perf_counter() - t0, self.P.solves - s0
        self.solves_per_apply = ns
        return dt, ns

    def time_ims(self):
        t0 = time.perf_counter()
        self.P.apply_A(self.r)
        return time.perf_counter() - t0

    def run_solves(self, quota):
        """Run BSP apply stages (one S application each, in apply order, a new
        apply starting when one completes) until >= quota solves: (solves, s)."""
        s0, t0 = self.P.solves, time.perf_counter()
        while self.P.solves - s0 < quota:
            if self._stages is None:
                self._stages = self.pc.bsp_apply_iter(self.r)
            try:
                next(self._stages)
            except StopIteration:
                self._stages = None
        return self.P.solves - s0, time.perf_counter() - t0


def cpu_baseline(cfgno, blocks=None):
    """The reference arithmetic on all host cores, bounded sample: one full BSP
    apply and one (I-S) apply after the shared-factor setup (~10-30 s at cfg5)."""
    ref = ReferenceCPU(cfgno, blocks=blocks)
    try:
        t_bsp, ns = ref.time_apply()
        t_ims = ref.time_ims()
    finally:
        ref.close()
    its, _ = reference_iterations(cfgno, blocks)
    per = t_bsp * ref.R
    out = {"value": 1.0 / per, "unit": "applies/s", "cores": ref.workers, "kind": "port",
           "sample": f"one full BSP apply ({ns} subdomain SuperLU solves + outgoing traces through the reference "
                     f"loop; x{ref.R} right-hand sides, the reference has one) and one (I-S) apply on "
                     f"{ref.workers} processes",
           "t_bsp_apply_s": t_bsp, "t_ims_apply_s": t_ims, "setup_s": ref.setup_s, "host": host_info()}
    if its:
        out["gmres_projected_s"] = ref.R * (its * (t_bsp + t_ims) + t_bsp)
        out["gmres_projection"] = (f"{its} reference iterations x (BSP + (I-S) apply) + the final x = M(V y) apply"
                                   + (f", x {ref.R} right-hand sides" if ref.R > 1 else ""))
    return out


def run_reference(args):
    """--impl reference: the reference path on the host cores (ReferenceCPU)."""
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    if rank != 0:
        return 0
    ref = ReferenceCPU(args.config, blocks=args.blocks)
    try:
        t_apply, ns = ref.time_apply()  # the first (warm-up) apply also sizes the samples
        t_ims = ref.time_ims()
        for _ in range(max(0, args.warmup - 1)):
            if t_apply * args.warmup > 60.0:
                break
            t_apply, ns = ref.time_apply()
        # each timed step is a bounded sample: a whole apply when the run fits in
        # ~2 minutes, otherwise the next S applications of the apply sequence up
        # to a solve quota (stage granularity; applies continue across steps)
        frac = min(1.0, 120.0 / max(1e-9, args.steps * t_apply))
        quota = max(1, int(round(frac * ns)))
        done, times = 0, []
        for _ in range(args.steps):
            k, dt = ref.run_solves(quota)
            done += k
            times.append(dt)
    finally:
        ref.close()
    wall = sum(times)
    value = (done / (ns * ref.R)) / wall
    its, t_golden = reference_iterations(args.config, args.blocks)
    c = ref.c
    cpu = {"value": value, "unit": "applies/s", "cores": ref.workers, "kind": "port",
           "sample": (f"each step: {'one full BSP apply' if frac >= 1.0 else f'{quota} of the {ns} subdomain solves of a BSP apply'}"
                      f" through the reference loop (S applications in apply order, gather / zero-skip / SuperLU "
                      f"solve / outgoing traces / scatter), every S application's solves on {ref.workers} forked "
                      f"processes" + (f"; x{ref.R} single-RHS applies per multi-RHS apply" if ref.R > 1 else "")),
           "setup_s": ref.setup_s, "t_bsp_apply_s": t_apply, "t_ims_apply_s": t_ims, "host": host_info()}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "applies/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(1, len(times)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "config": config_json(c, 1), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "applies/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if its:
        line["gmres"] = {"time_to_solution_s": ref.R * (its * (t_apply + t_ims) + t_apply), "projected": True,
                         "iterations": its,
                         "projection": "reference iterations x (BSP apply + (I-S) apply) + the final M apply, each "
                                       "timed above on this host" + (f", x {ref.R} right-hand sides" if ref.R > 1 else ""),
                         "build_container_measured_s": t_golden}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--blocks", type=int, default=None,
                    help="sweep block count p (BASELINE config 2 varies p over 1, 2, 4, 8; SURVEY.md §8d window rule)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the shared-operator variant")
    ap.add_argument("--no-peer", action="store_true",
                    help="row bands (N > 1): per-step kernels + NCCL send/recv instead of the fused apply over CUDA IPC")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import ctypes as C
    import torch
    from paper_2209_10886_b200 import native
    from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig

    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [native.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    c, spec, part = problem(args.config, args.blocks)
    R = int(c["nrhs"])
    sweep = SweepConfig(blocks=c["blocks"])
    torch.zeros(1, device=f"cuda:{local}")  # CUDA context up before the setup clock starts
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    system = GpuInterfaceSystem(spec, part, device=local, rank=rank, nranks=world, nccl_id=nccl_id, sweep=sweep)
    setup_s = time.perf_counter() - t0  # first factorisation: includes allocations and kernel loads
    peer = world > 1 and R == 1 and not args.no_peer
    if peer:
        system.enable_peer_memory()
    warm = []
    for _ in range(3):  # the same factorisation again (warm), median of three
        t0 = time.perf_counter()
        system.ctx.call("hs_factor")
        torch.cuda.synchronize()
        warm.append(time.perf_counter() - t0)
    setup_warm_s = sorted(warm)[1]
    L = system.layout.size
    gen = torch.Generator(device="cpu").manual_seed(1234)
    shape = (L,) if R == 1 else (L, R)
    r_host = torch.complex(torch.randn(shape, generator=gen, dtype=torch.float64),
                           torch.randn(shape, generator=gen, dtype=torch.float64))

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def measure(sysm, steps, warmup, with_clocks):
        """Device-resident BSP applies, CUDA events on the library stream."""
        ctx = sysm.ctx
        r = r_host.cuda()
        z = torch.empty_like(r)
        torch.cuda.synchronize()
        stream = torch.cuda.ExternalStream(ctx.stream())
        ctx.call("hs_set_async", 1)

        def apply_dev():
            ctx.call("hs_precond", native.HS_PC_BSP, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()), R,
                     native.HS_MEM_DEVICE)

        for _ in range(max(warmup, 3)):
            apply_dev()
        ctx.call("hs_sync")
        barrier()
        torch.cuda.synchronize()
        clocks = Clocks(local) if with_clocks else None
        if clocks:
            time.sleep(0.25)
        # the timed region: no per-launch events inside the library (they would
        # sit between the per-step launches of the multi-launch paths)
        l0 = ctx.launches()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            apply_dev()
        ev1.record(stream)
        ev1.synchronize()
        launches = ctx.launches() - l0
        clk = clocks.stop() if clocks else None
        barrier()
        torch.cuda.synchronize()
        ms = max_over_ranks(ev0.elapsed_time(ev1))
        # kernel durations for the roofline: the same applies again, each library
        # launch bracketed by events on the library stream
        nstat = min(steps, 50)
        ctx.kernel_stats(reset=True)
        ctx.call("hs_set_kernel_timing", 1)
        for _ in range(nstat):
            apply_dev()
        ctx.call("hs_sync")
        ctx.call("hs_set_kernel_timing", 0)
        kl, kms, kbytes, kflops = ctx.kernel_stats(reset=True)
        scale = steps / nstat  # per-step stats scaled to the timed region's step count
        kl, kms, kbytes, kflops = int(round(kl * scale)), kms * scale, kbytes * scale, kflops * scale
        # events around each of many short launches inflate their durations; the
        # kernels of a step cannot take longer than the step
        kms = min(kms, ms)
        ctx.call("hs_set_async", 0)
        return {"ms_per": ms / steps, "ms": ms, "launches": launches, "clk": clk, "kl": kl, "kms": kms,
                "kbytes": kbytes, "kflops": kflops}

    def gmres_tts(sysm):
        if R == 1:
            b = sysm.rhs()
        else:
            from paper_2209_10886_b200.configs import angles
            b = sysm.rhs(directions=[(float(np.cos(t)), float(np.sin(t))) for t in angles(c)])
        sysm.gmres(b, "bsp", tol=c["tol"], maxit=1000)  # warm (workspace allocation)
        runs = []
        for _ in range(3):  # median of three full solves
            barrier()
            t1 = time.perf_counter()
            res = sysm.gmres(b, "bsp", tol=c["tol"], maxit=1000)
            runs.append(max_over_ranks(time.perf_counter() - t1))  # synchronous call: host time brackets the device work
        tts = sorted(runs)[1]
        its = res.iterations if R == 1 else max(res.iterations)
        conv = res.converged if R == 1 else all(res.converged)
        out = {"time_to_solution_s": tts, "runs_s": runs, "iterations": its, "converged": bool(conv),
               "buffers": "host (numpy b in, numpy x out: the reference's interface)"}
        if world == 1:
            # the same solve with b and x resident in HBM (torch tensors through the same call)
            bd = torch.from_numpy(np.ascontiguousarray(b)).to(f"cuda:{local}")
            sysm.gmres(bd, "bsp", tol=c["tol"], maxit=1000)
            dr = []
            for _ in range(3):
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                sysm.gmres(bd, "bsp", tol=c["tol"], maxit=1000)
                torch.cuda.synchronize()
                dr.append(time.perf_counter() - t1)
            out["device_resident_s"] = sorted(dr)[1]
        if world == 1:  # with row bands each rank holds only its own blocks of x
            resid = np.linalg.norm(sysm.apply_interface_operator(res.solution) - b, axis=0) / np.linalg.norm(b, axis=0)
            out["true_relative_residual"] = float(np.max(resid))
        return out

    m = measure(system, args.steps, args.warmup, True)
    ms_per = m["ms_per"]
    value = 1e3 / ms_per
    share = m["kms"] / m["ms"] if m["ms"] > 0 else None
    if R == 1:
        # roofline of the HBM-bound step-apply kernel (per-subdomain maps)
        peak, peak_kind = load_peaks()
        ach = (m["kbytes"] / (m["kms"] * 1e-3)) / 1e9 if m["kms"] > 0 else None
        traffic, traffic_src = None, None
        prof = os.path.join(ROOT, "profiles", f"ncu_step_kernel_cfg{args.config}.json")
        if os.path.exists(prof) and m["kl"] > 0:
            with open(prof) as f:
                pj = json.load(f)
            # ncu DRAM bytes / algorithmic bytes of the captured launches, applied to
            # this run's average launch (the same per-launch unit as `achieved`)
            traffic = pj["traffic_over_algorithmic"] * m["kbytes"] / m["kl"]
            traffic_src = (f"profiles/{os.path.basename(prof)}: dram/algorithmic = "
                           f"{pj['traffic_over_algorithmic']:.4f} over {len(pj['launches'])} captured launches")
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": (ach / peak) if ach else None, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": ("k_bsp_tma, map-once plan (the whole BSP apply as one dataflow launch; maps staged "
                           "by TMA bulk copies with an L2 evict-first policy into an mbarrier ring; producer warp "
                           "+ 8 consumer warps + signaller warp; per-subdomain maps)") if m["kl"] <= args.steps else
                          "k_step1 (batched step-apply ZGEMV, per-subdomain maps)",
                "algorithmic_bytes_note": "bytes the map-once plan must move: 16 (rows cols + nv cols + 2 rows) per "
                                          "item (DESIGN.md 3a); SURVEY 8d's literal two-pass B_BSP is larger "
                                          "(15.84 GB at cfg5)",
                "peak_source": peak_kind,
                "peak_note": "measured peak = torch copy (half writes); this kernel's traffic is ~98% reads, so "
                             "frac can exceed 1 slightly; vs the 8 TB/s nominal HBM3e see achieved/8000",
                "launches": m["kl"], "kernel_ms_share_of_step": share,
                "algorithmic_bytes_per_apply": m["kbytes"] / max(args.steps, 1)}
    else:
        peak = fp64_peak()
        ach = (m["kflops"] / (m["kms"] * 1e-3)) / 1e12 if m["kms"] > 0 else None
        roof = {"bound": "fp64", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": (ach / peak) if ach else None, "traffic": None,
                "kernel": "k_zmma2_df (the whole R-RHS BSP apply as one persistent dataflow launch: FP64 DMMA m8n8k4, 3M "
                          "complex product, map chunks staged by bulk copies into an mbarrier ring; flops counted "
                          "as 8 per complex multiply-add)",
                "peak_source": "measured DMMA m8n8k4 peak, profiles/fp64_peak_b200.json",
                "launches": m["kl"], "kernel_ms_share_of_step": share,
                "algorithmic_flops_per_apply": m["kflops"] / max(args.steps, 1)}

    # e2e through the C ABI with pinned host buffers
    ctx = system.ctx
    stream = torch.cuda.ExternalStream(ctx.stream())
    r_pin = torch.from_numpy(r_host.numpy().copy()).pin_memory()
    z_pin = torch.empty_like(r_pin).pin_memory()

    def apply_host():
        ctx.call("hs_precond", native.HS_PC_BSP, C.c_void_p(r_pin.data_ptr()), C.c_void_p(z_pin.data_ptr()), R,
                 native.HS_MEM_HOST)

    for _ in range(2):
        apply_host()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ke = max(3, args.steps // 3)
    e0.record(stream)
    for _ in range(ke):
        apply_host()
    e1.record(stream)
    e1.synchronize()
    ems = max_over_ranks(e0.elapsed_time(e1))
    sync_value = 1e3 * ke / ems
    # the serving form (hs_precond_batch through system.precondition_batch): a
    # batch of host vectors, vector i+1 copied in and i-1 copied out while i is
    # applied; every step still moves its full input and result over PCIe
    r_b = [r_pin, torch.from_numpy(r_host.numpy().copy()).pin_memory()]
    z_b = [z_pin, torch.empty_like(r_pin).pin_memory()]
    rs, zs = [r_b[i % 2] for i in range(ke)], [z_b[i % 2] for i in range(ke)]
    system.precondition_batch(rs[:2], out=zs[:2])  # warm (slots, streams)
    barrier()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    system.precondition_batch(rs, out=zs)  # synchronous: returns with every result on the host
    pipe_s = max_over_ranks(time.perf_counter() - t1)
    e2e = {"value": ke / pipe_s, "unit": "applies/s", "h2d_bytes_per_step": int(L * R * 16),
           "d2h_bytes_per_step": int(L * R * 16),
           "mode": f"pipelined host batch of {ke} vectors (precondition_batch / hs_precond_batch), host clock "
                   "around the synchronous call",
           "sync_value": sync_value,
           "sync_mode": "one synchronous hs_precond call per vector (H2D, apply, D2H), CUDA events"}

    gm = None
    variants = {}
    if not args.no_gmres:
        gm = gmres_tts(system)
        gm["setup_s"] = setup_s
    if world == 1 and not args.no_variants and c["n"] % 16 == 0:
        # shared-operator variant: class maps only, every step one DMMA contraction
        del system
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        sh = GpuInterfaceSystem(spec, part, device=local, sweep=sweep, maps="shared")
        sh_setup = time.perf_counter() - t0
        ms_sh = measure(sh, max(10, args.steps), args.warmup, False)
        fl = ms_sh["kflops"] / (ms_sh["kms"] * 1e-3) / 1e12 if ms_sh["kms"] > 0 else None
        variants["shared_maps"] = {
            "what": "generic subdomains share one 4n x 4n map (discretization.py:224-229); each sweep step is "
                    "one FP64 DMMA contraction (k_zmma2: bulk-copy staged, 3M product, flops counted as 8 per "
                    "complex multiply-add) with the map L2-resident",
            "applies_per_s": 1e3 / ms_sh["ms_per"], "ms_per_apply": ms_sh["ms_per"],
            "roofline": {"bound": "fp64", "achieved": fl, "peak": fp64_peak(), "unit": "TFLOP/s",
                         "frac": fl / fp64_peak() if fl else None},
            "setup_s": sh_setup, "gmres": None if args.no_gmres else gmres_tts(sh),
            "map_bytes": sh.ctx.memory()}
        del sh
        torch.cuda.empty_cache()
        if R == 1:
            # one compact map per (operator class, face set), aliased by every subdomain of that
            # kind: the same fused map-once kernel and bitwise the same result, the stream from L2
            t0 = time.perf_counter()
            kd = GpuInterfaceSystem(spec, part, device=local, sweep=sweep, maps="kinds")
            kd_setup = time.perf_counter() - t0
            ms_kd = measure(kd, max(10, args.steps), args.warmup, False)
            variants["kind_maps"] = {
                "what": "maps='kinds': one compact map per (operator class, face set), every subdomain's record "
                        "aliasing its kind's; the per-subdomain path's kernels and bitwise its result, the map "
                        "stream served from L2 (evict-last policy)",
                "applies_per_s": 1e3 / ms_kd["ms_per"], "ms_per_apply": ms_kd["ms_per"],
                "l2_stream_gbs": (ms_kd["kbytes"] / (ms_kd["kms"] * 1e-3)) / 1e9 if ms_kd["kms"] > 0 else None,
                "setup_s": kd_setup, "gmres": None if args.no_gmres else gmres_tts(kd),
                "device_bytes": kd.ctx.memory()}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.config, args.blocks)
        except Exception as e:  # report, do not fail the bench
            cpu = {"value": None, "unit": "applies/s", "cores": 1, "kind": "port", "sample": f"failed: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "applies/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
                "config": config_json(c, world, "fused apply over CUDA IPC peer memory (NVLink)" if peer
                                     else "per-step kernels + NCCL send/recv"), "roofline": roof,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": m["launches"], "clocks": m["clk"],
                "gmres": gm, "setup_s": setup_s, "setup_warm_s": setup_warm_s, "variants": variants}
        if R > 1:  # one apply covers all R right-hand sides (RHS-applies/s for cfg 4)
            line["rhs_applies_per_s"] = value * R
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def fp64_peak():
    p = os.path.join(ROOT, "profiles", "fp64_peak_b200.json")
    with open(p) as f:
        return float(json.load(f)["dmma_m8n8k4_tflops"])


if __name__ == "__main__":
    sys.exit(main())
