# Round-2 closing evidence (after the factorisation and multi-RHS Arnoldi work):
# bench lines of every config with the final defaults, the reference arm, the
# launch list of the default bench command, launch lists of one GMRES solve
# (cfg3, cfg4, cfg5), the factorisation's launch list and a full capture of its
# kernels, the factorisation phase times.
O=gpurun_out/r02c
mkdir -p $O
for c in 5 3 1 4; do timeout 900 python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err; echo "cfg$c rc=$?"; done
for p in 1 2 4 8; do timeout 900 python bench.py --config 2 --blocks $p > $O/bench_cfg2_p$p.json 2> $O/bench_cfg2_p$p.err; echo "cfg2 p$p rc=$?"; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_cfg5.json 2> $O/bench_reference_cfg5.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_cfg5.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-gmres --no-variants > $O/ncu_b5.log 2>&1; echo "bench launches rc=$?"
for k in 3 4 5; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/gmres_launches_cfg$k.csv python tools/gmres_profile.py $k > $O/ncu_g$k.log 2>&1; echo "gmres$k rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 1500 --csv --log-file $O/setup_launches_cfg5.csv python tools/setup_profile.py 5 > $O/ncu_s5.log 2>&1; echo "setup launches rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_gj_inv|k_gj_update|k_zgemm_dmma|k_formS" -s 40 -c 12 -o $O/prof_setup_cfg5 \
  python tools/setup_profile.py 5 > $O/ncu_setup5.log 2>&1; echo "ncu setup5 rc=$?"
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_cgsgR" -s 120 -c 4 -o $O/prof_cgsgR_cfg4 python tools/gmres_profile.py 4 > $O/ncu_cgsgR.log 2>&1; echo "ncu cgsgR rc=$?"
for c in 5 3 2; do HS_FACTOR_TIMING=1 timeout 300 python tools/setup_time.py $c > $O/setup_time_cfg$c.txt 2>&1; echo "setup time $c rc=$?"; done
timeout 120 tools/_bin/gjinv_bench_0_2 > $O/gjinv_bench.jsonl 2>&1; echo "gjinv rc=$?"
python tools/gmres_r_time.py 4 > $O/gmres_r_cfg4.txt 2>&1; HS_ARNOLDI_R=mgs python tools/gmres_r_time.py 4 > $O/gmres_r_cfg4_mgs.txt 2>&1; echo "gmres_r rc=$?"
