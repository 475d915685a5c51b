for c in 4 5; do
python tools/dmma_variants.py $c 1
for ks in 1 2 4; do python tools/dmma_variants.py $c 3 HS_ZMMA_FUSED_KS=$ks; done
done 2>&1 | grep '"cfg"'
