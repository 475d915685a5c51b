"""Warm factorisation time of one config (hs_factor, median of five) with the
phase times of HS_FACTOR_TIMING=1 on stderr.
    HS_FACTOR_TIMING=1 python tools/setup_time.py CFG [maps]"""
import sys
import time

import torch

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
maps = sys.argv[2] if len(sys.argv) > 2 else "subdomain"
c = CONFIGS[k]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]), maps=maps)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.ctx.call("hs_factor")
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print({"config": k, "maps": maps, "hs_factor_s": sorted(ts)[2], "all": [round(t, 4) for t in ts]})
