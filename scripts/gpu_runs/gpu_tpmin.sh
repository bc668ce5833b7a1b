# two-phase threshold 2^26 instead of 2^28: gain on narrow mixed-sign data at 1e8 terms vs the extra launch on wide data
mkdir -p gpurun_out/tpmin
P=gpurun_out/tpmin
python scripts/build_variants.py rtp27 > $P/build.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases n01,c4s,c3,c2 --rounds 3 default rtp27 > $P/time.log 2>&1
true
