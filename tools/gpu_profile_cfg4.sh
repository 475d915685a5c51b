# cfg4 (64 RHS) DMMA launches of one BSP apply in the per-step map-once form:
# duration, DMMA pipe and FP64 tensor-path utilisation per launch; then one
# full capture of a sweep step and of the residual step.
B="python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
$B > gpurun_out/plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__cluster_dim_x --clock-control none -k regex:"k_zmma|k_block_fill" -s 54 -c 18 --csv --log-file gpurun_out/launches_cfg4.csv $B > gpurun_out/ncu4.log 2>&1; echo "rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"k_zmma" -s 54 -c 1 -o gpurun_out/prof_zmma_sweep_cfg4 $B > gpurun_out/ncu4s.log 2>&1; echo "rc=$?"
ncu --set full --import-source on --clock-control none -k regex:"k_zmma" -s 62 -c 1 -o gpurun_out/prof_zmma_resid_cfg4 $B > gpurun_out/ncu4r.log 2>&1; echo "rc=$?"
