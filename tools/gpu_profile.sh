# launch list of the default bench command (cfg5) + full captures of the fused BSP kernel at cfg5 and cfg3
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg5.csv $B > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_bsp_fused|k_bsp_tma" -s 3 -c 1 -o gpurun_out/prof_fused_cfg5 $B > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
B3="python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
$B3 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bsp_fused|k_bsp_tma" -s 3 -c 1 -o gpurun_out/prof_fused_cfg3 $B3 > gpurun_out/ncu3.log 2>&1; echo "ncu3 rc=$?"
