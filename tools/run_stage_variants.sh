# TMA ring depth of the fused apply: 5 stages (2 CTAs/SM) vs 12 stages (1 CTA/SM), BSP apply ms per config
for c in ${CFGS:-5 3 2 1}; do for st in 5 12; do
  HS_TMA_STAGES=$st timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-gmres --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c stages=$st', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3), round(d['roofline']['achieved']))"
done; done
