# launch lists (gpu__time_duration, every kernel) of the default bench command (cfg5) and of cfg3
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $B > gpurun_out/ncu1.log 2>&1; echo "rc=$?"
B3="python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv $B3 > gpurun_out/ncu3.log 2>&1; echo "rc=$?"
