# code-size probe: the sum kernel without the one-slot fast path (smaller kernel) on wide / mixed data
mkdir -p gpurun_out/nofast
P=gpurun_out/nofast
python scripts/build_variants.py nofast nodisp > $P/build.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c3,n01,c4s --rounds 3 default nofast nodisp > $P/time.log 2>&1
true
