# programmatic dependent launch of the per-step DMMA contraction: cfg4 apply and shared-map cfg5 apply
for p in 1 0; do
  HS_ZMMA_PDL=$p timeout 300 python bench.py --config 4 --steps 200 --warmup 5 --no-cpu-baseline --no-gmres --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 pdl=$p', round(d['ms_per_step'],4), 'ms')"
  HS_ZMMA_PDL=$p timeout 300 python -c "
import sys, torch; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
from conftest import cvec, product_problem
from paper_2209_10886_b200.configs import CONFIGS
from paper_2209_10886_b200.interface_system import GpuInterfaceSystem, SweepConfig
c=CONFIGS[5]; spec,part=product_problem(c)
s=GpuInterfaceSystem(spec,part,maps='shared',sweep=SweepConfig(blocks=c['blocks']))
g=torch.from_numpy(cvec(1,s.layout.size)).cuda(); st=torch.cuda.ExternalStream(s.ctx.stream()); s.ctx.call('hs_set_async',1)
for _ in range(5): s.bsp_apply(g)
torch.cuda.synchronize(); a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(50): s.bsp_apply(g)
b.record(st); b.synchronize(); s.ctx.call('hs_set_async',0)
print('shared cfg5 pdl=$p', round(a.elapsed_time(b)/50,4), 'ms')
"
done
