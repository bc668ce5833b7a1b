mkdir -p gpurun_out/tp
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x --timeout 900 -k "two_phase" > gpurun_out/tp/test_tp.log 2>&1
timeout 2400 python scripts/two_phase_sweep.py --cases 48 --seed 3 > gpurun_out/tp/sweep2.log 2>&1
true
