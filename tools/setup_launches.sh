# launch list of one warm factorisation at cfg5 (per-kernel time shares)
cat > /tmp/fac.py <<'PY'
import sys, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
c = CONFIGS[int(sys.argv[1])]
spec, part = product_problem(c)
s = GpuInterfaceSystem(spec, part, sweep=SweepConfig(blocks=c["blocks"]))
torch.cuda.synchronize()
torch.cuda.profiler.start()
s.ctx.call("hs_factor")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
PY
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/setup_launches_cfg5.csv python /tmp/fac.py 5 > /dev/null 2>&1; echo rc=$?
