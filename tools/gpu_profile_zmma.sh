B="python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-gmres"
$B > gpurun_out/plain_z.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_zmma -s 26 -c 13 -o gpurun_out/prof_zmma2_cfg5 $B > gpurun_out/ncu_z.log 2>&1; echo "ncu rc=$?"
