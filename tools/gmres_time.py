"""GMRES time-to-solution and iterations on one config (3 solves, median),
with the Arnoldi variant given by the environment (HS_MGS1_BLOCK, ...).
    python tools/gmres_time.py CFG [arnoldi]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import golden, product_problem, relerr
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig

k = int(sys.argv[1])
mode = sys.argv[2] if len(sys.argv) > 2 else "auto"
c = CONFIGS[k]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
G = golden(f"cfg{k}")
b = torch.from_numpy(np.asarray(G["b"])).cuda()
ts = []
for _ in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = s.gmres(b, "bsp", tol=1e-6, maxit=1000, arnoldi=mode)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
x = res.solution.cpu().numpy() if hasattr(res.solution, "cpu") else res.solution
h = np.array(res.history)
gh = np.asarray(G["gm_hist"])
n = min(len(h), len(gh))
out = {"config": k, "arnoldi": mode, "env": {kk: v for kk, v in os.environ.items() if kk.startswith("HS_")},
       "iterations": res.iterations, "golden_iterations": int(G["gm_iters"]), "time_s": sorted(ts[1:])[1],
       "x_vs_golden": relerr(x, G["gm_x"]), "hist_maxrel_vs_golden": float(np.max(np.abs(h[:n] - gh[:n]) / gh[:n]))}
if "acc_hist" in G.files:
    ah = np.asarray(G["acc_hist"]); n = min(len(h), len(ah))
    out["hist_maxrel_vs_accurate"] = float(np.max(np.abs(h[:n] - ah[:n]) / ah[:n]))
    out["x_vs_accurate"] = relerr(x, G["gm_x"] + G["acc_dx"])
print(json.dumps(out), flush=True)
