"""Per-tile timeline of one fused BSP apply (hs_set_trace): where a tile's
life goes (waiting for inputs / streaming its map / epilogue + signal), how
many CTAs stream at a time, and the tail.  One JSON line per config.
  python tools/fused_trace.py CFG [ims]"""
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
c = CONFIGS[cfg]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
g = torch.from_numpy(cvec(1, s.layout.size)).cuda()
for _ in range(3):
    s.bsp_apply(g)
s.ctx.call("hs_set_trace", 1)
s.bsp_apply(g)
torch.cuda.synchronize()
rows = C.c_int(0)
s.ctx.call("hs_get_trace", None, 0, C.byref(rows))
buf = (C.c_uint64 * (6 * rows.value))()
s.ctx.call("hs_get_trace", buf, rows.value, C.byref(rows))
s.ctx.call("hs_set_trace", 0)
tr = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 6)
t0 = tr[:, 0].min()
claim, start, ready, streamed, end = [(tr[:, i] - t0).astype(np.float64) / 1e3 for i in range(5)]
phase = (tr[:, 5] & 0xFF).astype(int)
cta = ((tr[:, 5] >> 8) & 0xFFFFFF).astype(int)
span = end.max()
out = {"config": cfg, "tiles": int(len(tr)), "ctas": int(len(set(cta))), "max_cta": int(cta.max()),
       "sms": int(len(set((tr[:, 5] >> 32).tolist()))), "span_us": round(span, 1),
       "claim_to_start_us": round(float(np.mean(start - claim)), 2),
       "wait_us": round(float(np.mean(ready - start)), 2), "stream_us": round(float(np.mean(streamed - ready)), 2),
       "epi_us": round(float(np.mean(end - streamed)), 2)}
# per CTA: time between finishing one tile and starting the next
gaps = []
for k in set(cta):
    m = np.where(cta == k)[0]
    o = m[np.argsort(start[m])]
    gaps.extend((start[o[1:]] - end[o[:-1]]).tolist())
out["gap_between_tiles_us"] = round(float(np.mean(gaps)), 2) if gaps else None
out["gap_p90_us"] = round(float(np.percentile(gaps, 90)), 2) if gaps else None
ph = {}
for p in sorted(set(phase)):
    m = phase == p
    ph[int(p)] = {"tiles": int(m.sum()), "wait": round(float(np.mean(ready[m] - start[m])), 2),
                  "stream": round(float(np.mean(streamed[m] - ready[m])), 2),
                  "first_start": round(float(start[m].min()), 1), "last_end": round(float(end[m].max()), 1)}
out["phases"] = ph
edges = np.linspace(0, span, 21)
st, busy = [], []
for a, b in zip(edges[:-1], edges[1:]):
    ov = np.clip(np.minimum(streamed, b) - np.maximum(ready, a), 0, None)
    st.append(round(float(ov.sum() / (b - a)), 1))
    ov2 = np.clip(np.minimum(end, b) - np.maximum(start, a), 0, None)
    busy.append(round(float(ov2.sum() / (b - a)), 1))
out["streaming_ctas_by_twentieth"] = st
out["working_ctas_by_twentieth"] = busy
print(json.dumps(out))
