import sys, time, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
c = CONFIGS[5]
spec, part = product_problem(c)
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
t0 = time.perf_counter()
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
torch.cuda.synchronize(); print("create+factor", time.perf_counter() - t0, "setup_time", s.setup_time)
for i in range(8):
    t0 = time.perf_counter(); s.ctx.call("hs_factor"); torch.cuda.synchronize(); print("refactor", i, time.perf_counter() - t0)
