timeout 900 python -m pytest tests/test_gpu_dmma.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/pt_dmma.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt_dmma.log
timeout 300 python bench.py --config 4 --no-cpu-baseline --no-gmres > gpurun_out/b4.json 2>gpurun_out/b4.err; echo "b4 rc=$?"
timeout 300 python bench.py --config 5 --no-cpu-baseline --no-gmres > gpurun_out/b5.json 2>gpurun_out/b5.err; echo "b5 rc=$?"
python - <<'PY'
import json
for f in ["gpurun_out/b4.json","gpurun_out/b5.json"]:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], d["roofline"]["frac"], "shared:", d["variants"]["shared_maps"]["ms_per_apply"], d["variants"]["shared_maps"]["roofline"]["frac"])
PY
B="python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-gmres --no-variants"
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__cluster_dim_x --clock-control none -k regex:"k_zmma|k_block_fill" -s 54 -c 18 --csv --log-file gpurun_out/launches_cfg4.csv $B > gpurun_out/ncu4.log 2>&1; echo "rc=$?"
