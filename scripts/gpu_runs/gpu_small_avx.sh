# config 1 after the AVX-512 small-accumulator path: bench lines (both arms) + C-loop probe on the box's CPU
mkdir -p gpurun_out/small
P=gpurun_out/small
for r in 1 2; do
timeout 600 python bench.py --config 1 > $P/bench_c1_$r.json 2>&1
timeout 600 python bench.py --config 1 --impl reference > $P/ref_c1_$r.json 2>&1
done
g++ -O2 scripts/probes/small_exact_sum.cpp -o /tmp/small_probe -ldl && /tmp/small_probe $PWD/oracle/_ref/libexsum_ref.so $PWD/paper_1505_05571_b200/lib/libexsum_b200.so > $P/c_loop.log 2>&1
grep -m1 -o "avx512f" /proc/cpuinfo >> $P/c_loop.log
true
