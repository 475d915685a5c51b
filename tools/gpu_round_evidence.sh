# Round evidence: bench lines for every config + the reference arm, launch lists
# and full ncu captures of the fused apply (cfg5, cfg3), GMRES launch lists.
for c in 5 3 2 1 4; do timeout 900 python bench.py --config $c > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo "cfg$c rc=$?"; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $B > gpurun_out/ncu1.log 2>&1; echo "launches5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bsp_fused|k_bsp_tma" -s 3 -c 1 -o gpurun_out/prof_fused_cfg5 $B > gpurun_out/ncu2.log 2>&1; echo "full5 rc=$?"
B3="python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv $B3 > gpurun_out/ncu3l.log 2>&1; echo "launches3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bsp_fused|k_bsp_tma" -s 3 -c 1 -o gpurun_out/prof_fused_cfg3 $B3 > gpurun_out/ncu3.log 2>&1; echo "full3 rc=$?"
for k in 5 3; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gmres_launches_cfg$k.csv python tools/gmres_profile.py $k > gpurun_out/ncu_g$k.log 2>&1; echo "gmres$k rc=$?"
done
for c in 5 3 2; do timeout 300 python tools/fused_trace.py $c > gpurun_out/trace_cfg$c.json 2>/dev/null; echo "trace$c rc=$?"; done
