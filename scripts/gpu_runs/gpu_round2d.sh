mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2d_gpu_tests.log 2>&1
for i in 1 2; do
python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2d_c5_defer_$i.json 2>&1
EXSUM_LIB=paper_1505_05571_b200/lib/variants/seg_nodefer.so python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2d_c5_nodefer_$i.json 2>&1
done
python scripts/e2e_probe.py --threads 16,15,14 > gpurun_out/r2d_e2e_probe.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench_c4.json 2> gpurun_out/r2d_bench_c4.err
true
