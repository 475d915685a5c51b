# Round-2 final evidence: bench lines with the final defaults, the reference
# arm, launch lists of one GMRES solve (cfg3, cfg5), ncu captures of the DMMA
# dataflow kernel and of the one-reduction Arnoldi kernels.
mkdir -p gpurun_out/r02b
for c in 5 3 1 4; do timeout 900 python bench.py --config $c > gpurun_out/r02b/bench_cfg$c.json 2> gpurun_out/r02b/bench_cfg$c.err; echo "cfg$c rc=$?"; done
for p in 1 2 4 8; do timeout 900 python bench.py --config 2 --blocks $p > gpurun_out/r02b/bench_cfg2_p$p.json 2> gpurun_out/r02b/bench_cfg2_p$p.err; echo "cfg2 p$p rc=$?"; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02b/bench_reference_cfg5.json 2> gpurun_out/r02b/bench_reference_cfg5.err; echo "ref rc=$?"
for k in 3 5; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b/gmres_launches_cfg$k.csv python tools/gmres_profile.py $k > gpurun_out/r02b/ncu_g$k.log 2>&1; echo "gmres$k rc=$?"
done
B4="python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_zmma2_df" -s 3 -c 1 -o gpurun_out/r02b/prof_zmma2_df_cfg4 $B4 > gpurun_out/r02b/ncu4.log 2>&1; echo "ncu df rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_cgsg" -s 120 -c 4 -o gpurun_out/r02b/prof_cgsg_cfg3 python tools/gmres_profile.py 3 > gpurun_out/r02b/ncu_cgsg.log 2>&1; echo "ncu cgsg rc=$?"
timeout 120 python tools/zmma_df_trace.py 4 64 > gpurun_out/r02b/zmma2_df_trace_cfg4.json 2>&1; echo "trace rc=$?"
# factorisation kernels and the MGS Arnoldi kernels (profiles/r02/ncu_setup_cfg3.json, ncu_mgs1*.json)
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_gj_inv|k_gj_update|k_zgemm_dmma|k_formS" -c 12 -o gpurun_out/r02b/prof_setup_cfg3 \
  python tools/setup_profile.py 3 > gpurun_out/r02b/ncu_setup3.log 2>&1; echo "ncu setup3 rc=$?"
for k in 3 2; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_mgs1" -s 5 -c 3 -o gpurun_out/r02b/prof_mgs_cfg$k \
    python tools/gmres_profile_mode.py $k mgs > gpurun_out/r02b/ncu_mgs$k.log 2>&1; echo "ncu mgs$k rc=$?"
done
