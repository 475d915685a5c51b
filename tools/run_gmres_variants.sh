for cfg in 3 5; do
python tools/gmres_variants.py $cfg grid
for pf in 0 1 2; do python tools/gmres_variants.py $cfg auto HS_MGS1_PF=$pf; done
done 2>&1 | grep config
