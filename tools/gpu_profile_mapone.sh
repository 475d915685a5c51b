# map-once fused BSP apply: bench lines (cfg5, cfg3), launch list of the default
# bench command, full ncu captures of the fused kernel at cfg5 and cfg3
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench5 rc=$?"
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench3 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg5.csv $B > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bsp_fused|k_bsp_tma" -s 3 -c 1 -o gpurun_out/prof_fused_cfg5 $B > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
B3="python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg3.csv $B3 > gpurun_out/ncu3l.log 2>&1; echo "ncu3l rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bsp_fused|k_bsp_tma" -s 3 -c 1 -o gpurun_out/prof_fused_cfg3 $B3 > gpurun_out/ncu3.log 2>&1; echo "ncu3 rc=$?"
