import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import product_problem, cvec
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
R = int(sys.argv[2]) if len(sys.argv) > 2 else 40
spec, part = product_problem(CONFIGS[k])
s = GpuInterfaceSystem(spec, part)
X = cvec(3, s.layout.size, R)
Y = s.apply_interface_operator(X); print("ims ok", flush=True)
Z = s.bj_half_apply(X, "forward"); print("fwd ok", flush=True)
Z = s.bsp_apply(X); print("bsp ok", flush=True)
