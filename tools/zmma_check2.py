"""Where a multi-RHS forward sweep differs from the single-RHS one: per
32-column chunk of right-hand sides and per block (diagnostics)."""
import sys

import numpy as np

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import cvec, product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig

c = CONFIGS[int(sys.argv[1])]
R = int(sys.argv[2])
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
L, n = s.layout.size, c["n"]
X = cvec(3, L, R)
F = s.forward_sweep(X)
ref = np.stack([s.forward_sweep(np.ascontiguousarray(X[:, r])) for r in range(R)], 1)
d = np.abs(F - ref)
bad = d > 1e-10 * np.abs(ref).max()
print("bad elements", int(bad.sum()), "of", bad.size)
cols = np.where(bad.any(0))[0]
print("bad RHS columns", cols.tolist()[:100])
blocks = np.where(bad.reshape(-1, n, R).any((1, 2)))[0]
print("bad blocks (1-based m)", (blocks + 1).tolist()[:60])
rows = np.where(bad.reshape(-1, n, R).any((0, 2)))[0]
print("bad positions within block", rows.tolist()[:70])
