# per-warp dispatch of the one-slot fast path (EXSUM_UNIFORM_DISPATCH)
mkdir -p gpurun_out/disp
P=gpurun_out/disp
timeout 900 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py tests/test_products.py tests/test_property.py -m gpu -q -x --timeout 600 > $P/tests.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c4,c3,c2 --rounds 4 default nodisp nofast > $P/time.log 2>&1
true
