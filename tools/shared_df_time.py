"""Shared-map (maps="shared") BSP apply and GMRES per fused mask: per-step
k_zmma2 launches (mask 3) vs the dataflow launch (mask 11 = bit 3), ms per
apply (CUDA events, device buffers), kernel flops per apply, the result's
difference to mask 3, GMRES time and iterations.
    python tools/shared_df_time.py CFG [MASK ...]"""
import ctypes as C
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import cvec, product_problem, relerr
from paper_2209_10886_b200 import native
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
masks = [int(m) for m in sys.argv[2:]] or [3, 11]
c = CONFIGS[k]
spec, part = product_problem(c)
peak = json.load(open("profiles/fp64_peak_b200.json"))["dmma_m8n8k4_tflops"]
ref = None
for mask in masks:
    s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]), maps="shared", fused=mask)
    ctx = s.ctx
    r = torch.from_numpy(cvec(3, s.layout.size)).cuda()
    z = torch.empty_like(r)
    stream = torch.cuda.ExternalStream(ctx.stream())

    def apply_dev():
        ctx.call("hs_precond", native.HS_PC_BSP, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()), 1,
                 native.HS_MEM_DEVICE)

    ctx.call("hs_set_async", 1)
    for _ in range(5):
        apply_dev()
    ctx.call("hs_sync")
    torch.cuda.synchronize()
    n = 100
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        apply_dev()
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    ctx.kernel_stats(reset=True)
    ctx.call("hs_set_kernel_timing", 1)
    apply_dev()
    ctx.call("hs_sync")
    ctx.call("hs_set_kernel_timing", 0)
    kl, kms, kbytes, kflops = ctx.kernel_stats(reset=True)
    ctx.call("hs_set_async", 0)
    zz = z.cpu().numpy()
    if ref is None:
        ref = zz
    b = s.rhs()
    s.gmres(b, "bsp", tol=c["tol"], maxit=1000)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        res = s.gmres(b, "bsp", tol=c["tol"], maxit=1000)
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"config": k, "mask": mask, "ms_per_apply": ms, "launches_per_apply": kl,
                      "kernel_gflop_per_apply": kflops / 1e9,
                      "frac_dmma_peak_on_kernel_flops": kflops / (ms * 1e-3) / 1e12 / peak,
                      "rel_diff_vs_first": relerr(zz, ref), "gmres_s": sorted(ts)[1],
                      "iterations": res.iterations}), flush=True)
    del s
    torch.cuda.empty_cache()
