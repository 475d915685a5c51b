B="python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-gmres"
$B > gpurun_out/plain_z.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_zmma -s 30 -c 2 -o gpurun_out/prof_zmma_cfg5 $B > gpurun_out/ncu_z.log 2>&1; echo "ncu rc=$?"
B4="python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
$B4 > gpurun_out/plain_z4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_zmma -s 30 -c 2 -o gpurun_out/prof_zmma_cfg4 $B4 > gpurun_out/ncu_z4.log 2>&1; echo "ncu rc=$?"
