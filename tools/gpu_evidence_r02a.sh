# Round-2 evidence A: compute-sanitizer over the dataflow kernels, ncu captures of
# the factorisation and Arnoldi kernels.  Every command is bounded by timeout.
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  for case in tma fused zmma gmres; do
    env=""
    [ "$case" = "fused" ] && env="HS_FUSED_TMA=0"
    log=gpurun_out/sanitize_${tool}_${case}.log
    timeout 420 env $env compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_case.py $case > $log 2>&1
    echo "$tool $case rc=$?" | tee -a gpurun_out/sanitize_summary.txt
    tail -4 $log
  done
done
python tools/setup_profile.py 3 > gpurun_out/setup3.log 2>&1; echo "setup3 rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_gj_inv|k_gj_update|k_zgemm_dmma|k_formS" -c 12 -o gpurun_out/prof_setup_cfg3 \
  python tools/setup_profile.py 3 > gpurun_out/ncu_setup3.log 2>&1; echo "ncu setup3 rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/setup_launches_cfg5.csv python tools/setup_profile.py 5 > gpurun_out/ncu_setup5.log 2>&1; echo "setup5 launches rc=$?"
for k in 3 2; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_mgs1" -s 5 -c 3 -o gpurun_out/prof_mgs_cfg$k \
    python tools/gmres_profile.py $k > gpurun_out/ncu_mgs$k.log 2>&1; echo "ncu mgs$k rc=$?"
done
