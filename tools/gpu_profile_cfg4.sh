# cfg4 (64 RHS) DMMA launches of one BSP apply in the per-step map-once form:
# duration, DMMA pipe and FP64 tensor-path utilisation per launch
B="python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
$B > gpurun_out/plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:"k_zmma|k_block_fill" -s 54 -c 18 --csv --log-file gpurun_out/launches_cfg4.csv $B > gpurun_out/ncu4.log 2>&1; echo "rc=$?"
