# ripple build: L2 prefetch distance 0 (the batch the refills load next) vs 1
mkdir -p gpurun_out/pf0
P=gpurun_out/pf0
python scripts/build_variants.py rpf0 > $P/build.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c2,c3,c5,c4 --rounds 3 default rpf0 > $P/time.log 2>&1
true
