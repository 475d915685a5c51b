# Round 2: fresh full captures of the fused HBM apply (k_bsp_tma) at cfg5 and
# cfg3 with the launch lists of the same commands, for
# profiles/ncu_step_kernel_cfg{5,3}.json (bench.py's roofline.traffic).
O=gpurun_out/r02e
mkdir -p $O
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv $B > $O/ncu1.log 2>&1; echo "launches5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bsp_fused|k_bsp_tma" -s 3 -c 1 -o $O/prof_fused_cfg5 $B > $O/ncu2.log 2>&1; echo "full5 rc=$?"
B3="python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv $B3 > $O/ncu3l.log 2>&1; echo "launches3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bsp_fused|k_bsp_tma" -s 3 -c 1 -o $O/prof_fused_cfg3 $B3 > $O/ncu3.log 2>&1; echo "full3 rc=$?"
for c in 5 3; do timeout 300 python tools/fused_trace.py $c > $O/fused_trace_cfg$c.json 2>/dev/null; echo "trace$c rc=$?"; done
