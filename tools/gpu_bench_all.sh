# full bench lines (defaults: CPU baseline, GMRES, variants) for every config + the reference arm at cfg5
for c in 5 3 2 1 4; do python bench.py --config $c > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "cfg$c rc=$?"; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
