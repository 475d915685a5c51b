# map-once plan: BSP apply ms per config, kernel (TMA / register) x ticket order (list-scheduled / plan order)
for c in ${CFGS:-5 3 2 1}; do for t in ${TMAS:-0 1}; do for o in ${ORDERS:-1 0}; do
  HS_FUSED_TMA=$t HS_FUSED_ORDER=$o timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-gmres --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c tma=$t order=$o', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3), round(d['roofline']['achieved']))"
done; done; done
