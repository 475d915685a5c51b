"""Map-once vs per-step fused plan: z difference, BSP apply time and GMRES
A M v time for one config (device vectors, CUDA events).  One JSON line.
  python tools/map_once_check.py CFG"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem, cvec, relerr
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig

cfg = int(sys.argv[1])
c = CONFIGS[cfg]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
g = torch.from_numpy(cvec(1, s.layout.size)).cuda()
st = torch.cuda.ExternalStream(s.ctx.stream())


def timed(fn, N):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        for _ in range(N):
            fn()
        b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / N


out = {"config": cfg}
N = 20 if cfg == 5 else 50
res = {}
for plan, mask in (("steps", 5), ("map_once", 1)):
    s.ctx.call("hs_set_fused", mask)
    z = s.bsp_apply(g)
    res[plan] = z.cpu().numpy()
    out[plan + "_ms"] = round(timed(lambda: s.bsp_apply(g), N), 4)
    r = s.gmres(s.rhs(), "bsp", tol=1e-6, maxit=1000)
    r = s.gmres(s.rhs(), "bsp", tol=1e-6, maxit=1000)
    out[plan + "_gmres"] = [r.iterations, float(r.history[-1]), round(r.wall_time, 4)]
    out[plan + "_x"] = r.solution
out["z_relerr"] = relerr(res["map_once"], res["steps"])
out["x_relerr"] = relerr(out.pop("map_once_x"), out.pop("steps_x"))
print(json.dumps(out))
