import sys, numpy as np, subprocess
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
if len(sys.argv) == 1:
    for n in (16, 32, 48, 64, 128):
        for R in (2, 8, 40):
            for lat in ((2, 2), (4, 4)):
                p = subprocess.run([sys.executable, __file__, str(n), str(R), str(lat[0]), str(lat[1])], capture_output=True, text=True)
                print(n, R, lat, p.stdout.strip().splitlines()[-1] if p.stdout.strip() else ("FAIL " + p.stderr.strip().splitlines()[-1]), flush=True)
    sys.exit(0)
from conftest import product_problem, cvec, relerr
from paper_2209_10886_b200.configs import small_case
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem
n, R, a, b = map(int, sys.argv[1:5])
c = small_case(a, b, n, kappa=2 * np.pi * n / 20)
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part)
X = cvec(3, s.layout.size, R)
Y = s.apply_interface_operator(X)
e = max(relerr(Y[:, r], s.apply_interface_operator(np.ascontiguousarray(X[:, r]))) for r in range(R))
print("ok", e)
