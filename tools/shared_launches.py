"""A few BSP applies of the shared-map variant (for an ncu launch list)."""
import sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import cvec, product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = CONFIGS[cfg]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, maps="shared", sweep=SweepConfig(blocks=c["blocks"]))
g = torch.from_numpy(cvec(1, s.layout.size)).cuda()
for _ in range(3):
    s.bsp_apply(g)
torch.cuda.synchronize()
torch.cuda.profiler.start()
s.bsp_apply(g)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
