"""Per-CTA timeline of the per-step DMMA contraction (k_zmma2, hs_set_trace):
for every launch of one BSP apply (R right-hand sides, or the shared maps)
the CTA count, the launch's span, the gap after the previous launch, and
where a CTA's time goes: setup (task + column tables, ring init), waiting for
its first chunk, the contraction, split-K reduction + epilogue.
  python tools/zmma_trace.py CFG [R] [shared]"""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import cvec, product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig

cfg = int(sys.argv[1])
R = int(sys.argv[2]) if len(sys.argv) > 2 else 64
maps = "shared" if "shared" in sys.argv[3:] else "subdomain"
c = CONFIGS[cfg]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, maps=maps, fused=False, sweep=SweepConfig(blocks=c["blocks"]))
g = torch.from_numpy(cvec(1, s.layout.size, R) if R > 1 else cvec(1, s.layout.size)).cuda()
for _ in range(3):
    s.bsp_apply(g)
torch.cuda.synchronize()
s.ctx.call("hs_set_trace", 1)
s.bsp_apply(g)
torch.cuda.synchronize()
rows = C.c_int(0)
s.ctx.call("hs_get_trace", None, 0, C.byref(rows))
buf = (C.c_uint64 * (6 * rows.value))()
s.ctx.call("hs_get_trace", buf, rows.value, C.byref(rows))
s.ctx.call("hs_set_trace", 0)
tr = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 6).astype(np.int64)
t0 = tr[:, 0].min()
seq = tr[:, 5] >> 40
out = {"config": cfg, "R": R, "maps": maps, "rows": int(len(tr)), "launches": []}
prev_end = None
tot = 0.0
for q in sorted(set(seq.tolist())):
    m = seq == q
    t = (tr[m, :5] - t0) / 1e3
    full = t[:, 3] > 0  # rows with a contraction record (rank 0 and others)
    span = t[:, 4].max() - t[:, 0].min()
    rec = {"ctas": int(m.sum()), "start": round(float(t[:, 0].min()), 2), "span_us": round(float(span), 2),
           "gap_us": None if prev_end is None else round(float(t[:, 0].min() - prev_end), 2),
           "setup": round(float(np.mean(t[:, 1] - t[:, 0])), 2),
           "first_chunk": round(float(np.mean(t[full, 2] - t[full, 1])), 2),
           "contract": round(float(np.mean(t[full, 3] - t[full, 2])), 2),
           "tail": round(float(np.mean(t[full, 4] - t[full, 3])), 2),
           "cta_us_max": round(float(np.max(t[:, 4] - t[:, 0])), 2),
           "start_spread": round(float(t[:, 0].max() - t[:, 0].min()), 2)}
    prev_end = t[:, 4].max()
    out["launches"].append(rec)
out["apply_span_us"] = round(float((tr[:, 4].max() - t0) / 1e3), 1)
print(json.dumps(out))
