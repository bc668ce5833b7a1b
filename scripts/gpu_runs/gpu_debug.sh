mkdir -p gpurun_out/debug
P=gpurun_out/debug
export EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/debug.so
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests_debug.log 2>&1
timeout 600 python scripts/sanitize_run.py > $P/sanitize_run.log 2>&1
for c in 4 5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $P/bench_c$c.json 2>&1; done
true
