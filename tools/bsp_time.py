"""Time the 1-RHS BSP apply (device-resident vectors, CUDA events) for one
config; knobs via environment (HS_FUSED_TMA, HS_FUSED_NW): one JSON line.
  python tools/bsp_time.py CFG [ENV=VAL ...]"""
import json, os, sys
for kv in sys.argv[2:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem, cvec
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
cfg = int(sys.argv[1])
c = CONFIGS[cfg]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
g = torch.from_numpy(cvec(1, s.layout.size)).cuda()
out = torch.empty_like(g)
for _ in range(5):
    s.bsp_apply(g)
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(s.ctx.stream())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 50 if cfg != 5 else 20
with torch.cuda.stream(st):
    a.record(st)
    for _ in range(N):
        s.bsp_apply(g)
    b.record(st)
b.synchronize()
ms = a.elapsed_time(b) / N
ref = s.bsp_apply(g)
print(json.dumps({"config": cfg, "env": sys.argv[2:], "ms_per_apply": round(ms, 4), "checksum": [float(ref.real.sum()), float(ref.imag.sum())]}))
