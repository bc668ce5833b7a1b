# segmented: claim-order histogram over the tail only + one-load-per-thread scan
mkdir -p gpurun_out/emit
P=gpurun_out/emit
timeout 900 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py tests/test_context_gpu.py -m gpu -q -x --timeout 600 > $P/tests2.log 2>&1
FB_R=7 FB_CASES=segmented timeout 600 python scripts/flat_bound.py >> $P/time2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c5_2.csv python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c5_2.log 2>&1
true
