# round 2, second session: final evidence on the final build (driver commands + per-config lines + config-5 ncu)
mkdir -p gpurun_out/final5
P=gpurun_out/final5
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/ref.json 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench.json 2> $P/bench.err
for c in 2 3 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $P/bench_c$c.json 2> $P/bench_c$c.err; done
timeout 600 python bench.py --impl reference --config 5 --steps 20 --warmup 5 > $P/ref_c5.json 2>&1
timeout 600 python bench.py --config 1 > $P/bench_c1.json 2>&1
timeout 600 python bench.py --config 1 --impl reference > $P/ref_c1.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"exsum_segment" -s 4 -c 4 -o $P/r02_c5b python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c5.log 2>&1
for c in 4 5; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c$c.csv python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c$c.log 2>&1; done
true
