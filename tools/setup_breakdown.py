import sys, time
t00 = time.perf_counter()
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem
from paper_2209_10886_b200 import native
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.discretization import ImpedanceSpec, scatterer_cells
t0 = time.perf_counter()
torch.cuda.init(); torch.cuda.synchronize()
t1 = time.perf_counter()
c = CONFIGS[5]; spec, part = product_problem(c)
imp = ImpedanceSpec.for_problem(spec)
ctx = native.Context(0, part.n1, part.n2, spec.cells_per_side, spec.h, spec.kappa, complex(imp.coefficient), 0, 1)
t2 = time.perf_counter()
home, cells = scatterer_cells(spec, part)
cc = native.i32(cells)
ctx.call("hs_set_dirichlet", home.i1, home.i2, native.iptr(cc), len(cc))
t3 = time.perf_counter()
ctx.call("hs_factor"); torch.cuda.synchronize()
t4 = time.perf_counter()
ctx.call("hs_factor"); torch.cuda.synchronize()
t5 = time.perf_counter()
print(f"imports {t0-t00:.3f} cuda_init {t1-t0:.3f} create {t2-t1:.3f} dirichlet {t3-t2:.3f} factor_cold {t4-t3:.3f} factor_warm {t5-t4:.3f}")
