import sys, time, ctypes as C
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem, cvec
from paper_2209_10886_b200 import native
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
c = CONFIGS[5]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
L = s.layout.size
ctx = s.ctx
st = torch.cuda.ExternalStream(ctx.stream())
hp = torch.from_numpy(cvec(1, L)).pin_memory(); zp = torch.empty_like(hp).pin_memory()
d = hp.cuda(); dz = torch.empty_like(d)
def ev(): return torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    for name, fn in [("h2d", lambda: d.copy_(hp, non_blocking=True)), ("d2h", lambda: zp.copy_(d, non_blocking=True))]:
        fn(); torch.cuda.synchronize()
        a, b = ev(), ev(); a.record(st)
        for _ in range(10): fn()
        b.record(st); b.synchronize(); print(name, "ms", a.elapsed_time(b) / 10, "GB/s", 16 * L / (a.elapsed_time(b) / 10 * 1e-3) / 1e9)
def run(mem, src, dst):
    ctx.call("hs_precond", native.HS_PC_BSP, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()), 1, mem)
for mem, src, dst, nm in [(native.HS_MEM_DEVICE, d, dz, "device"), (native.HS_MEM_HOST, hp, zp, "host")]:
    run(mem, src, dst); torch.cuda.synchronize()
    t0 = time.perf_counter(); a, b = ev(), ev(); a.record(st)
    for _ in range(10): run(mem, src, dst)
    b.record(st); b.synchronize(); t1 = time.perf_counter()
    print(nm, "event ms", a.elapsed_time(b) / 10, "wall ms", (t1 - t0) * 100)
