# segmented: next-segment head prefetch variant vs default
mkdir -p gpurun_out/pfnext
P=gpurun_out/pfnext
python scripts/build_variants.py rpfnext > $P/build.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c5 --rounds 4 default rpfnext > $P/time.log 2>&1
true
