mkdir -p gpurun_out
for C in 1 2 4; do echo "== copies $C"; taskset -c 2 ./scripts/probes/host_kernel_c$C 50000000; done > gpurun_out/r2_host_kernel.log 2>&1
python scripts/host_rates.py --n 2e8 > gpurun_out/r2_host_rates2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r2_gpu_tests.log 2>&1
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref_c4.json 2> gpurun_out/r2_ref_c4.err
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err
true
