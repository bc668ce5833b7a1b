# ripple knobs: segmented split / vectors per lane / prefetch distance / warps
mkdir -p gpurun_out/ripple2
P=gpurun_out/ripple2
python scripts/build_variants.py ripple rsplit rseg8 rseg6 rv7 rpf2 rw10 rsegfix0 > $P/build.log 2>&1
timeout 2400 python scripts/ab_variants.py --cases c3,c5,c2 --rounds 3 default ripple rsplit rseg8 rseg6 rv7 rpf2 rw10 rsegfix0 > $P/time.log 2>&1
true
