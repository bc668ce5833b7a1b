# round 2, fourth session: last check of the final tree (kernels as in gpu_final8.sh; probe knobs compiled out)
mkdir -p gpurun_out/final9
P=gpurun_out/final9
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/ref.json 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench.json 2> $P/bench.err
for c in 3 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $P/bench_c$c.json 2> $P/bench_c$c.err; done
true
