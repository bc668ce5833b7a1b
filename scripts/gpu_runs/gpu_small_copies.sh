mkdir -p gpurun_out/smallc
cd scripts/probes
for i in 1 2; do for v in default small1 small4 small8; do
  if [ $v = default ]; then L=../../paper_1505_05571_b200/lib/libexsum_b200.so; else L=../../paper_1505_05571_b200/lib/variants/$v.so; fi
  echo "== $v" >> ../../gpurun_out/smallc/small.log
  taskset -c 3 ./small_bench $L >> ../../gpurun_out/smallc/small.log 2>&1
done; done
true
