# plain sums: vectors per lane per batch on narrow and wide data (ripple build); product kernels on the new defaults
mkdir -p gpurun_out/vsum
P=gpurun_out/vsum
python scripts/build_variants.py rv4 rv5 ripplev6 rv7 > $P/build.log 2>&1
timeout 2400 python scripts/ab_variants.py --cases c1,n01,c2,c3,c4s --rounds 3 default rv7 ripplev6 rv5 rv4 > $P/time.log 2>&1
python scripts/time_products.py > $P/products.log 2>&1
timeout 900 python -m pytest tests/test_products.py tests/test_property.py -m gpu -q > $P/tests.log 2>&1
true
