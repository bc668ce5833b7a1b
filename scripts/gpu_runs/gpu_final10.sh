# round 2, fourth session: the final tree (sqnorm / dot batch sizes changed since gpu_final9.sh)
mkdir -p gpurun_out/final10
P=gpurun_out/final10
python scripts/build_variants.py debug > $P/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/ref.json 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench.json 2> $P/bench.err
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/debug.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests_debug.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/debug.so timeout 600 python scripts/sanitize_run.py > $P/sanitize_debug.log 2>&1
timeout 400 python scripts/long_sweep.py --seconds 240 --seed 41 > $P/long_sweep.log 2>&1
true
