# sqnorm / dot: vectors per lane per batch on the ripple build
mkdir -p gpurun_out/products2
P=gpurun_out/products2
python scripts/build_variants.py sq3 sq4 sq5 dot2 dot3 > $P/build.log 2>&1
for v in default sq3 sq4 sq5 dot2 dot3; do
  echo "== $v" >> $P/time.log
  if [ $v = default ]; then python scripts/time_products.py >> $P/time.log 2>&1; else EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/$v.so python scripts/time_products.py >> $P/time.log 2>&1; fi
done
true
