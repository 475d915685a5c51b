"""Factorise one config twice (the second call is warm: no module loading) and
print both setup times -- also the program profiled for the setup kernels."""
import sys, time
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
c = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
torch.cuda.synchronize()
t0 = time.perf_counter()
s.ctx.call("hs_factor")
torch.cuda.synchronize()
print("setup_s first", round(s.setup_time, 4), "warm", round(time.perf_counter() - t0, 4))
