"""The dataflow DMMA apply (fused mask bit 1: k_zmma2_df) against the per-step
form (k_zmma2) on R right-hand sides: result agreement and ms per apply.
    python tools/zmma_df_check.py CFG R [reps]"""
import json
import sys
import time

import numpy as np
import torch

sys.path[:0] = [".", "tests"]
from conftest import cvec, product_problem, relerr  # noqa: E402
from paper_2209_10886_b200.configs import CONFIGS  # noqa: E402
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig  # noqa: E402

cfg, R = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
c = CONFIGS[cfg]
spec, part = product_problem(c)
out = {"config": cfg, "R": R}
X = torch.from_numpy(cvec(5, spec and GpuInterfaceSystem(spec, part, device=-1).layout.size, R)).cuda()
res = {}
for name, mask in (("per_step", 1), ("dataflow", 3)):
    s = GpuInterfaceSystem(spec, part, fused=mask, sweep=SweepConfig(blocks=c["blocks"]))
    Z = s.bsp_apply(X)
    for _ in range(3):
        s.bsp_apply(X)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        Z = s.bsp_apply(X)
    torch.cuda.synchronize()
    out[f"{name}_ms"] = (time.perf_counter() - t0) * 1e3 / reps
    res[name] = Z.cpu().numpy()
    if name == "dataflow":
        z1 = s.bsp_apply(np.ascontiguousarray(X[:, 0].cpu().numpy()))
        out["dataflow_col0_vs_single"] = relerr(res[name][:, 0], z1)
        Z2 = s.bsp_apply(X).cpu().numpy()
        out["dataflow_repeat_bitwise"] = bool(np.array_equal(Z2, res[name]))
    del s
out["dataflow_vs_per_step"] = relerr(res["dataflow"], res["per_step"])
print(json.dumps(out), flush=True)
