"""A/B of the host-buffer BSP apply (hs_precond, pinned buffers, one sync per
call): HS_IO_OVERLAP=1 (chunked transfers overlapped with the kernel) vs 0.
  python tools/e2e_ab.py CFG  -> one JSON line per run"""
import json, os, subprocess, sys
if len(sys.argv) > 2:  # worker
    import ctypes as C, time
    import torch
    sys.path.insert(0, "."); sys.path.insert(0, "tests")
    from conftest import product_problem, cvec
    from paper_2209_10886_b200 import native
    from paper_2209_10886_b200.configs import CONFIGS
    from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
    c = CONFIGS[int(sys.argv[1])]
    spec, part = product_problem(c)
    s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
    hp = torch.from_numpy(cvec(1, s.layout.size)).pin_memory(); zp = torch.empty_like(hp).pin_memory()
    run = lambda: s.ctx.call("hs_precond", native.HS_PC_BSP, C.c_void_p(hp.data_ptr()), C.c_void_p(zp.data_ptr()), 1, native.HS_MEM_HOST)
    for _ in range(5): run()
    N = 60 if int(sys.argv[1]) != 5 else 30
    t0 = time.perf_counter()
    for _ in range(N): run()
    dt = (time.perf_counter() - t0) / N
    print(json.dumps({"cfg": int(sys.argv[1]), "overlap": os.environ.get("HS_IO_OVERLAP"), "ms_per_call": dt * 1e3}))
    sys.exit(0)
for rep in range(3):
    for io in ("1", "0"):
        out = subprocess.run([sys.executable, __file__, sys.argv[1], "w"], env=dict(os.environ, HS_IO_OVERLAP=io),
                             capture_output=True, text=True).stdout.strip().splitlines()
        print(out[-1] if out else "{}")
