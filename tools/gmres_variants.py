"""Time full GMRES solves (CUDA events around hs_gmres, no profiler) for the
Arnoldi variants; one JSON line per (config, variant).  Variant knobs are
environment variables read once per process, so each variant runs in its own
process: python tools/gmres_variants.py CFG ARNOLDI [ENV=VAL ...]."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
for kv in sys.argv[3:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
from conftest import product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
cfg, mode = int(sys.argv[1]), sys.argv[2]
c = CONFIGS[cfg]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
b = torch.from_numpy(s.rhs()).cuda()
ts = []
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = s.gmres(b, "bsp", tol=1e-6, maxit=1000, arnoldi=mode)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(json.dumps({"config": cfg, "arnoldi": mode, "env": sys.argv[3:], "iterations": r.iterations,
                  "tts_s": sorted(ts[1:])[1], "all": ts}))
