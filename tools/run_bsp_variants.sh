# bench.py apply numbers (device-resident, CUDA events) per fused-kernel variant
for c in ${CFGS:-1 2 3 5}; do
for v in "HS_FUSED_TMA=0" "HS_FUSED_TMA=0 HS_FUSED_NW=8" "HS_FUSED_TMA=1 HS_FUSED_NW=8 HS_TMA_STAGES=5" "HS_FUSED_TMA=1 HS_FUSED_NW=8 HS_TMA_STAGES=3"; do
env $v python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-gmres --no-variants 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('cfg', $c, '$v', 'ms/step', round(d['ms_per_step'],4), 'frac', round(d.get('roofline',{}).get('frac'),3))"
done; done
