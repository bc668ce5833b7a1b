mkdir -p gpurun_out/il
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/interleave.so timeout 900 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py tests/test_property.py tests/test_products.py tests/test_p2p.py -m gpu -q -x --timeout 600 > gpurun_out/il/tests.log 2>&1
for i in 1 2 3; do TV_OVERLAP=1 TV_CONFIGS=2,3,4,6 python scripts/time_variants.py interleave >> gpurun_out/il/time.log 2>&1; done
true
