# Arnoldi kernels timed with CUDA events (no profiler), L = cfg3 and cfg5 interface sizes
for L in 122880 499712; do ./tools/mgs_bench $L 60 | grep -v exchange; done
