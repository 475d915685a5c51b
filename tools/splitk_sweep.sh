# split-K variants of the fused apply (HS_SPLITK) and of the DMMA dataflow (HS_ZMMA2_SPLIT)
for c in 3 5 2; do for m in 0 1 2; do
HS_SPLITK=$m timeout 120 python bench.py --config $c --steps 100 --no-cpu-baseline --no-gmres --no-variants > gpurun_out/sk.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/sk.json').read().strip().splitlines()[-1]); print('cfg$c HS_SPLITK=$m', round(d['ms_per_step'],4))"
done; done
for m in 0 1; do
HS_ZMMA2_SPLIT=$m timeout 120 python bench.py --config 4 --steps 100 --no-cpu-baseline --no-gmres --no-variants > gpurun_out/sk.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/sk.json').read().strip().splitlines()[-1]); print('cfg4 HS_ZMMA2_SPLIT=$m', round(d['ms_per_step'],4))"
done
