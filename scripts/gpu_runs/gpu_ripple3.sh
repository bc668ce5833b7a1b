# ripple as the default build: GPU suite (with the carry-chain test), ncu of configs 3 and 5, benches
mkdir -p gpurun_out/ripple3
P=gpurun_out/ripple3
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
for c in 3 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $P/bench_c$c.json 2> $P/bench_c$c.err; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exsum_sum_kernel -s 3 -c 1 -o $P/r02_c3_ripple python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"exsum_segmented_kernel" -s 3 -c 1 -o $P/r02_c5_ripple python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c5.log 2>&1
true
