# completion signalling of the TMA fused kernel: signaller warp (0) vs consumers directly (1)
for c in ${CFGS:-5 3 2 1}; do for d in 0 1; do
  HS_DIRECT_SIGNAL=$d timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline --no-gmres --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c direct=$d', round(d['ms_per_step'],4), 'ms', round(d['roofline']['frac'],3))"
done; done
