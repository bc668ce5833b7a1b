# ripple + software-pipelined decode (EXSUM_RIPPLE_PIPE): A/B and GPU suite under the variant
mkdir -p gpurun_out/pipe
P=gpurun_out/pipe
python scripts/build_variants.py rpipe rpipev7 > $P/build.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c3,c5,n01,c2 --rounds 3 default rpipe rpipev7 > $P/time.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/rpipe.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > $P/tests.log 2>&1
true
