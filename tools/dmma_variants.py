"""Time the 64-RHS BSP apply (cfg4) and the shared-map 1-RHS apply (cfg5) with
per-step DMMA launches (fused=1) or the fused DMMA dataflow kernel (fused=3);
split-K of the fused kernel via HS_ZMMA_FUSED_KS.  python tools/dmma_variants.py CFG FUSED [ENV=VAL]"""
import json, os, sys
for kv in sys.argv[3:]:
    k, v = kv.split("=", 1); os.environ[k] = v
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem, cvec
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
cfg, fused = int(sys.argv[1]), int(sys.argv[2])
c = CONFIGS[cfg]
spec, part = product_problem(c)
maps = "shared" if cfg == 5 else "subdomain"
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]), maps=maps, fused=fused)
R = 64 if cfg == 4 else 1
g = torch.from_numpy(cvec(3, s.layout.size, None if R == 1 else R)).cuda()
for _ in range(3): s.bsp_apply(g)
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(s.ctx.stream())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 20
a.record(st)
for _ in range(N): z = s.bsp_apply(g)
b.record(st); b.synchronize()
print(json.dumps({"cfg": cfg, "fused": fused, "env": sys.argv[3:], "ms": a.elapsed_time(b) / N,
                  "check": float(torch.view_as_real(z).abs().sum())}))
