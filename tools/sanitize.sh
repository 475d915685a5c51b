# compute-sanitizer over the dataflow kernels (run on the GPU box):
#   bash tools/sanitize.sh  -> gpurun_out/sanitize_<tool>_<case>.log
# memcheck: out-of-bounds / misaligned global and shared accesses;
# racecheck: shared-memory hazards (mbarrier rings, DSMEM exchanges);
# synccheck: illegal barrier / warp-sync use.  Each run is bounded by timeout.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for case in tma fused zmma gmres; do
    env=""
    [ "$case" = "fused" ] && env="HS_FUSED_TMA=0"
    log=gpurun_out/sanitize_${tool}_${case}.log
    timeout 900 env $env compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_case.py $case > $log 2>&1
    echo "$tool $case rc=$?" | tee -a gpurun_out/sanitize_summary.txt
    tail -3 $log
  done
done
