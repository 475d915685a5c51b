B="python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
$B > gpurun_out/plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:"k_zmma" -s 51 -c 17 --csv --log-file gpurun_out/launches_cfg4.csv $B > gpurun_out/ncu4.log 2>&1; echo "rc=$?"
