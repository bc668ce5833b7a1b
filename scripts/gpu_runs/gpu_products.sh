# sqnorm / dot timing on the ripple build vs the slot layout and vs fewer vectors per lane
mkdir -p gpurun_out/products
P=gpurun_out/products
python scripts/build_variants.py noripple rv4 rv5 rv7 ripplev6 > $P/build.log 2>&1
for v in default noripple rv7 ripplev6 rv5 rv4; do
  echo "== $v" >> $P/time.log
  if [ $v = default ]; then python scripts/time_products.py >> $P/time.log 2>&1; else EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/$v.so python scripts/time_products.py >> $P/time.log 2>&1; fi
done
true
