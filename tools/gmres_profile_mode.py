"""One GMRES solve with a given Arnoldi mode bracketed by cudaProfilerStart/Stop
(ncu --profile-from-start off).  python tools/gmres_profile_mode.py CFG MODE"""
import sys
import torch
sys.path[:0] = [".", "tests"]
from conftest import product_problem  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402
k, mode = int(sys.argv[1]), sys.argv[2]
c = CONFIGS[k]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
b = s.rhs()
s.gmres(b, "bsp", tol=1e-6, maxit=1000, arnoldi=mode)
torch.cuda.synchronize()
torch.cuda.profiler.start()
res = s.gmres(b, "bsp", tol=1e-6, maxit=1000, arnoldi=mode)
torch.cuda.profiler.stop()
print("iterations", res.iterations)
