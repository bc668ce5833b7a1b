mkdir -p gpurun_out/final2
P=gpurun_out/final2
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/ref.json 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench.json 2> $P/bench.err
timeout 600 python bench.py --config 1 > $P/bench_c1.json 2>&1
timeout 600 python bench.py --config 1 --impl reference > $P/ref_c1.json 2>&1
true
