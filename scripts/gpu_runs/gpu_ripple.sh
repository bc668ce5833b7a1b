# ripple variant (two unsigned 32-bit-word planes, 12 warps per SM): GPU suite under EXSUM_LIB, A/B timing
mkdir -p gpurun_out/ripple
P=gpurun_out/ripple
python scripts/build_variants.py ripple ripplev6 > $P/build.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/ripple.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > $P/tests.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c3,c5,c2,c4 --rounds 3 default ripple ripplev6 > $P/time.log 2>&1
true
