O=gpurun_out/r02d
mkdir -p $O
timeout 900 python bench.py --config 4 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 120 python tools/zmma_df_trace.py 4 64 > $O/zmma2_df_trace_cfg4.json 2>&1; echo "trace rc=$?"
B4="python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_zmma2_df" -s 3 -c 1 -o $O/prof_zmma2_df_cfg4 $B4 > $O/ncu4.log 2>&1; echo "ncu df rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/gmres_launches_cfg4.csv python tools/gmres_profile.py 4 > $O/ncu_g4.log 2>&1; echo "gmres4 rc=$?"
