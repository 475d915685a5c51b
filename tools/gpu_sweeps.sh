# Measured-and-rejected variants (DESIGN.md §3a / §6): split-K pairs of the
# fused apply (HS_SPLITK=1 all strips, 2 critical path only) and of the DMMA
# dataflow (HS_ZMMA2_SPLIT), L2 prefetch of a tile's later chunks
# (HS_TMA_PREFETCH=1 whole rest, 2 one ring).  One line per variant.
line() { python -c "import json,sys; d=json.loads(open('gpurun_out/sw.json').read().strip().splitlines()[-1]); print(sys.argv[1], round(d['ms_per_step'],4))" "$1"; }
for c in 3 5 2; do for m in 0 1 2; do
  HS_SPLITK=$m timeout 120 python bench.py --config $c --steps 100 --no-cpu-baseline --no-gmres --no-variants > gpurun_out/sw.json 2>/dev/null; line "cfg$c HS_SPLITK=$m"
done; done
for m in 0 1; do
  HS_ZMMA2_SPLIT=$m timeout 120 python bench.py --config 4 --steps 100 --no-cpu-baseline --no-gmres --no-variants > gpurun_out/sw.json 2>/dev/null; line "cfg4 HS_ZMMA2_SPLIT=$m"
done
for c in 3 5; do for pf in 0 1 2; do
  HS_TMA_PREFETCH=$pf timeout 120 python bench.py --config $c --steps 100 --no-cpu-baseline --no-gmres --no-variants > gpurun_out/sw.json 2>/dev/null; line "cfg$c HS_TMA_PREFETCH=$pf"
done; done
