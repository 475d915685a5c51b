# k_bsp_tma L2 prefetch of the chunks beyond the ring (HS_TMA_PREFETCH) on every config
for c in 3 5; do for pf in 0 2; do
HS_TMA_PREFETCH=$pf timeout 120 python bench.py --config $c --steps 200 --no-cpu-baseline --no-variants > gpurun_out/pf.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/pf.json').read().strip().splitlines()[-1]); print('cfg$c prefetch=$pf', round(d['ms_per_step'],4), 'gmres', round(d['gmres']['time_to_solution_s'],4))"
done; done
