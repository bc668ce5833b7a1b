# timing probe (wrong sums by construction): the ripple body at 16 warps per SM (one plane for both signs)
mkdir -p gpurun_out/t16
P=gpurun_out/t16
python scripts/build_variants.py t16v8 t16v6 t16v5 > $P/build.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c3,c5,n01 --rounds 3 default t16v8 t16v6 t16v5 > $P/time.log 2>&1
true
