import sys, numpy as np, subprocess
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
if len(sys.argv) == 1:
    for args in (["s", 64, 40, 8, 8], ["s", 64, 33, 8, 8], ["c", 2, 16], ["c", 2, 32], ["c", 2, 33], ["c", 2, 40], ["c", 2, 64], ["c", 1, 64]):
        p = subprocess.run([sys.executable, __file__] + [str(a) for a in args], capture_output=True, text=True)
        print(args, p.stdout.strip().splitlines()[-1] if p.stdout.strip() else ("FAIL " + p.stderr.strip().splitlines()[-1]), flush=True)
    sys.exit(0)
from conftest import product_problem, cvec, relerr
from paper_2209_10886_b200.configs import small_case, CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem
if sys.argv[1] == "s":
    n, R, a, b = map(int, sys.argv[2:6])
    c = small_case(a, b, n, kappa=2 * np.pi * n / 20)
else:
    c = CONFIGS[int(sys.argv[2])]; R = int(sys.argv[3])
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part)
X = cvec(3, s.layout.size, R)
Y = s.apply_interface_operator(X)
e = max(relerr(Y[:, r], s.apply_interface_operator(np.ascontiguousarray(X[:, r]))) for r in range(R))
print("ok", e)
