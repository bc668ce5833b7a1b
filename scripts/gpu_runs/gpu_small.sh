mkdir -p gpurun_out/small
timeout 900 python -m pytest tests/test_gpu.py tests/test_context_gpu.py tests/test_io.py tests/test_capi.py tests/test_benchrec.py -m gpu -q --timeout 600 > gpurun_out/small/tests.log 2>&1
python scripts/latency_probe.py > gpurun_out/small/latency.log 2>&1
true
