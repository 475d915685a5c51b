# bench apply lines (device + e2e) for configs 1 2 3 5, GMRES time-to-solution included
for c in 1 2 3 5; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | tail -1 > gpurun_out/b$c.json; done
python tools/bench_summary.py gpurun_out/b1.json gpurun_out/b2.json gpurun_out/b3.json gpurun_out/b5.json
