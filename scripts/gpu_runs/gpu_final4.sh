mkdir -p gpurun_out/final4
P=gpurun_out/final4
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/ref.json 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench.json 2> $P/bench.err
for c in 2 3; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $P/bench_c$c.json 2> $P/bench_c$c.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exsum_sum_kernel -s 3 -c 1 -o $P/r02_c4_il python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c4.csv python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c4.log 2>&1
true
