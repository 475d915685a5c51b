# Arnoldi kernels timed with CUDA events (no profiler); cluster slice sweep for k_mgs1c
for L in 1536 14336 32768; do for ch in 512 1024 2048 4096; do HS_MGS1C_CHUNK=$ch ./tools/mgs_bench $L 60 | grep k_mgs1c | sed "s/^/L=$L chunk<=$ch /"; done; done
