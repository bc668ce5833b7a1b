mkdir -p gpurun_out/hold
P=gpurun_out/hold
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -k "launch_config or golden" --timeout 300 > $P/tests.log 2>&1
timeout 600 python bench.py --config 4 --hold 5 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > $P/c4_hold5.json 2>&1
timeout 600 python bench.py --config 5 --hold 5 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > $P/c5_hold5.json 2>&1
timeout 600 python bench.py --config 2 --hold 5 --steps 1000 --warmup 5 --no-e2e --no-cpu-baseline > $P/c2_hold5.json 2>&1
true
