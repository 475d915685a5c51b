"""Per-task timeline of one dataflow DMMA apply (k_zmma2_df, hs_set_trace):
per phase the mean wait for inputs, slab latency, contraction and
epilogue+signal, the span, and how many CTAs contract at a time.
    python tools/zmma_df_trace.py CFG R [subdomain|shared]"""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path[:0] = [".", "tests"]
from conftest import cvec, product_problem  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

cfg, R = int(sys.argv[1]), int(sys.argv[2])
maps = sys.argv[3] if len(sys.argv) > 3 else "subdomain"
c = CONFIGS[cfg]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, fused=11 if maps == "shared" else 3, maps=maps,
                       sweep=SweepConfig(blocks=c["blocks"]))
X = torch.from_numpy(cvec(5, s.layout.size, R)).cuda()
for _ in range(3):
    s.bsp_apply(X)
torch.cuda.synchronize()
s.ctx.call("hs_set_trace", 1)
s.bsp_apply(X)
torch.cuda.synchronize()
rows = C.c_int(0)
s.ctx.call("hs_get_trace", None, 0, C.byref(rows))
buf = (C.c_uint64 * (6 * rows.value))()
s.ctx.call("hs_get_trace", buf, rows.value, C.byref(rows))
s.ctx.call("hs_set_trace", 0)
tr = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 6).astype(np.int64)
t0 = tr[:, 0].min()
claim, met, first, comp, sig = [(tr[:, i] - t0) / 1e3 for i in range(5)]
phase = tr[:, 5] & 0xFF
out = {"config": cfg, "R": R, "maps": maps, "tasks": int(len(tr)), "span_us": round(float(sig.max()), 1), "phases": {}}
for p in sorted(set(phase.tolist())):
    m = phase == p
    out["phases"][int(p)] = {"tasks": int(m.sum()), "wait_inputs": round(float(np.mean(met[m] - claim[m])), 2),
                             "slab_latency": round(float(np.mean(first[m] - met[m])), 2),
                             "contract": round(float(np.mean(comp[m] - first[m])), 2),
                             "epilogue_signal": round(float(np.mean(sig[m] - comp[m])), 2),
                             "first_claim": round(float(claim[m].min()), 1), "last_signal": round(float(sig[m].max()), 1)}
edges = np.linspace(0, sig.max(), 21)
out["contracting_ctas"] = [int(np.sum((first < b) & (comp > a))) for a, b in zip(edges[:-1], edges[1:])]
print(json.dumps(out))
