"""Factorisation (setup) of one config bracketed by cudaProfilerStart/Stop, for
ncu --profile-from-start off captures of k_gj_inv / k_gj_update / k_zgemm_dmma.

    python tools/setup_profile.py CFG
"""
import sys

import torch

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = CONFIGS[k]
spec, part = product_problem(c)
GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))  # warm (module load, workspace)
torch.cuda.synchronize()
torch.cuda.profiler.start()
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("setup done", s.layout.size)
