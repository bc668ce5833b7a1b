# robustness after the pipelined fix-up and the claim-order change: bounds-checked build through the GPU
# suite and the sanitize workload; 300 s randomized parity sweep on the default build
mkdir -p gpurun_out/robust
P=gpurun_out/robust
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/debug.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests_debug.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/debug.so timeout 600 python scripts/sanitize_run.py > $P/sanitize_debug.log 2>&1
timeout 500 python scripts/long_sweep.py --seconds 300 --seed 7 > $P/long_sweep.log 2>&1
true
