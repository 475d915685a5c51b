"""One GMRES solve bracketed by cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[k]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
if int(c["nrhs"]) > 1:  # config 4: one right-hand side per incident angle
    from paper_2209_10886_b200.configs import angles
    b = s.rhs(directions=[(float(np.cos(t)), float(np.sin(t))) for t in angles(c)])
else:
    b = s.rhs()
s.gmres(b, "bsp", tol=1e-6, maxit=1000)
torch.cuda.synchronize()
torch.cuda.profiler.start()
res = s.gmres(b, "bsp", tol=1e-6, maxit=1000)
torch.cuda.profiler.stop()
print("iterations", res.iterations if int(c["nrhs"]) == 1 else max(res.iterations))
