# round 2, second session: pipelined Inf/NaN fix-up in the segmented kernel (EXSUM_SEG_FIX_GROUP)
mkdir -p gpurun_out/segfix
P=gpurun_out/segfix
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
for v in default segfix2 segfix0; do
  if [ $v = default ]; then unset EXSUM_LIB; else export EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/$v.so; fi
  FB_R=7 FB_CASES=segmented,segmented_nospec timeout 600 python scripts/flat_bound.py >> $P/segfix_time.log 2>&1
done
unset EXSUM_LIB
FB_R=5 FB_CASES=flat,flat_nospec timeout 600 python scripts/flat_bound.py >> $P/segfix_time.log 2>&1
true
