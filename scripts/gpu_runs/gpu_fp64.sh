mkdir -p gpurun_out/fp64
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/fp64dec.so timeout 900 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py tests/test_property.py tests/test_products.py -m gpu -q -x --timeout 600 > gpurun_out/fp64/tests.log 2>&1
for i in 1 2; do TV_OVERLAP=1 TV_CONFIGS=2,3,4,6 python scripts/time_variants.py fp64dec >> gpurun_out/fp64/time.log 2>&1; done
true
