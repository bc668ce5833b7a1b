# confirm EXSUM_SEG_VEC=7 for the segmented kernel (5 interleaved rounds) + its tests
mkdir -p gpurun_out/resweep
P=gpurun_out/resweep
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/seg7.so timeout 900 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py tests/test_context_gpu.py -m gpu -q -x --timeout 600 -k "seg" > $P/tests_seg7.log 2>&1
timeout 1200 python scripts/ab_variants.py --cases c5 --rounds 5 default seg7 > $P/seg7_confirm.log 2>&1
true
