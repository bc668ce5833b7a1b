# round 2, fourth session: final evidence on the two-plane build (fresh container rebuild)
mkdir -p gpurun_out/final7
P=gpurun_out/final7
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/ref.json 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench.json 2> $P/bench.err
for c in 2 3 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $P/bench_c$c.json 2> $P/bench_c$c.err; done
for c in 4 5; do timeout 600 python bench.py --config $c --hold 5 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > $P/hold_c$c.json 2>&1; done
true
