# claim-ahead + register preload of the next head before the epilogue (EXSUM_SEG_AHEAD=2)
mkdir -p gpurun_out/segahead
P=gpurun_out/segahead
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/segahead3.so timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x --timeout 600 -k "seg" > $P/tests3.log 2>&1
for v in default segahead3; do
  if [ $v = default ]; then unset EXSUM_LIB; else export EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/$v.so; fi
  FB_R=7 FB_CASES=segmented timeout 600 python scripts/flat_bound.py >> $P/time3.log 2>&1
done
true
