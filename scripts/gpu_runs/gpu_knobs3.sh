# ripple build: grid policy for short overlapped sums and the segmented claim-order tail, re-checked at 12 warps
mkdir -p gpurun_out/knobs3
P=gpurun_out/knobs3
python scripts/build_variants.py fullgrid segtail2 segtail8 > $P/build.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c2,c3,n01,c5 --rounds 3 default fullgrid segtail2 segtail8 > $P/time.log 2>&1
true
