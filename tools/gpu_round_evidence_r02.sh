# Round-2 evidence: bench lines (every config, cfg2 block sweep), the reference
# arm, the cfg4 DMMA launch list and full captures of k_zmma2.
mkdir -p gpurun_out/r02
for c in 5 3 1 4; do timeout 900 python bench.py --config $c > gpurun_out/r02/bench_cfg$c.json 2> gpurun_out/r02/bench_cfg$c.err; echo "cfg$c rc=$?"; done
for p in 1 2 4 8; do timeout 900 python bench.py --config 2 --blocks $p > gpurun_out/r02/bench_cfg2_p$p.json 2> gpurun_out/r02/bench_cfg2_p$p.err; echo "cfg2 p$p rc=$?"; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02/bench_reference_cfg5.json 2> gpurun_out/r02/bench_reference_cfg5.err; echo "ref rc=$?"
B4="python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x --clock-control none -k regex:"k_zmma|k_block_fill" -s 54 -c 18 --csv --log-file gpurun_out/r02/launches_cfg4.csv $B4 > gpurun_out/r02/ncu4.log 2>&1; echo "ncu4 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_zmma2" -s 51 -c 9 -o gpurun_out/r02/prof_zmma2_cfg4 $B4 > gpurun_out/r02/ncu4f.log 2>&1; echo "ncu4 full rc=$?"
python tools/zmma_trace.py 4 64 > gpurun_out/r02/zmma_trace_cfg4.json 2>&1; echo "trace4 rc=$?"
python tools/zmma_trace.py 5 1 shared > gpurun_out/r02/zmma_trace_cfg5_shared.json 2>&1; echo "trace5 rc=$?"
