# GMRES launch list (one solve) for the configs given as arguments (default: 2 1)
for k in ${@:-2 1}; do
python tools/gmres_profile.py $k > gpurun_out/gp$k.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gmres_launches_cfg$k.csv python tools/gmres_profile.py $k > gpurun_out/ncu_g$k.log 2>&1; echo "rc=$?"
done
