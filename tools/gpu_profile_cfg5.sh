python -m pytest tests/test_gpu_scale.py -x -q 2>&1 | tail -25
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-gmres"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_step1|k_vec|k_mgs|k_givens" -c 100 --csv --log-file gpurun_out/launches_cfg5.csv $B > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_step1 -s 20 -c 3 -o gpurun_out/prof_step_cfg5 $B > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out
