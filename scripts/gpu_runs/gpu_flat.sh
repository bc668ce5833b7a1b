mkdir -p gpurun_out/flat
P=gpurun_out/flat
timeout 600 python scripts/flat_bound.py > $P/flat_bound2.log 2>&1
for v in segfix0 segfix1; do FB_CASES=segmented,segmented_nospec EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/$v.so timeout 600 python scripts/flat_bound.py >> $P/flat_bound2.log 2>&1; done
true
