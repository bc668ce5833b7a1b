# segmented: early claim atomic + (offsets, segment) claim records (EXSUM_SEG_CLAIM2)
mkdir -p gpurun_out/claim2
P=gpurun_out/claim2
timeout 900 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py tests/test_context_gpu.py -m gpu -q -x --timeout 600 > $P/tests.log 2>&1
for r in 1; do
for v in default es16 esinf claim3rt; do
  if [ $v = default ]; then unset EXSUM_LIB; else export EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/$v.so; fi
  FB_R=7 FB_CASES=segmented timeout 600 python scripts/flat_bound.py >> $P/time.log 2>&1
done
done
true
