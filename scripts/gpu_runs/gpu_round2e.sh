mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_context_gpu.py tests/test_benchrec.py tests/test_gpu.py -m gpu -q --timeout 600 -x > gpurun_out/r2e_gpu_tests.log 2>&1
timeout 600 python bench.py --config 5 --steps 20 --warmup 5 > gpurun_out/r2e_bench_c5.json 2> gpurun_out/r2e_bench_c5.err
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e_bench_c4.json 2> gpurun_out/r2e_bench_c4.err
true
