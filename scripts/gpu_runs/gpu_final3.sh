mkdir -p gpurun_out/final3
P=gpurun_out/final3
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/debug.so timeout 600 python scripts/sanitize_run.py > $P/sanitize_debug.log 2>&1
timeout 600 python scripts/sanitize_run.py > $P/sanitize_default.log 2>&1
true
