mkdir -p gpurun_out/segflat
P=gpurun_out/segflat
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x --timeout 600 -k "seg" > $P/tests6.log 2>&1
FB_CASES=segmented,flat timeout 600 python scripts/flat_bound.py > $P/time6.log 2>&1
for v in flatg0; do FB_CASES=segmented EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/$v.so timeout 600 python scripts/flat_bound.py >> $P/time6.log 2>&1; done
true
