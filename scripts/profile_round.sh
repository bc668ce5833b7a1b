set -x
mkdir -p gpurun_out/prof
for c in 2 3 4 5; do timeout 300 python bench.py --config $c > gpurun_out/prof/bench_c$c.json 2> gpurun_out/prof/bench_c$c.err; done
timeout 300 python bench.py --impl reference > gpurun_out/prof/bench_ref_c2.json 2>&1
timeout 300 python bench.py --impl reference --config 4 > gpurun_out/prof/bench_ref_c4.json 2>&1
for c in 2 3 4; do timeout 600 ncu --set full --clock-control none --import-source on -k regex:exsum_sum_kernel -s 3 -c 1 -o gpurun_out/prof/r01h_c$c python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu_c$c.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exsum_segmented_kernel -s 3 -c 1 -o gpurun_out/prof/r01h_c5 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu_c5.log 2>&1
for c in 2 3 4 5; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c$c.csv python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/launch_c$c.log 2>&1; done
ls -la gpurun_out/prof
