# cluster split-K depth of the per-step DMMA launches (PDL on, no per-launch events in the timed region)
for ks in 1 2 4 8; do
  HS_ZMMA_KS=$ks timeout 300 python bench.py --config 4 --steps 200 --warmup 5 --no-cpu-baseline --no-gmres --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 ks=$ks', round(d['ms_per_step'],4), 'ms')"
done
