mkdir -p gpurun_out/segsplit
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/segsplit.so timeout 900 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py tests/test_context_gpu.py -m gpu -q -x --timeout 600 > gpurun_out/segsplit/tests.log 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['roofline']['kernel_ms'], d['value'])" >> gpurun_out/segsplit/var.log 2>&1
  EXSUM_LIB=paper_1505_05571_b200/lib/variants/segsplit.so timeout 300 python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('segsplit', d['roofline']['kernel_ms'], d['value'])" >> gpurun_out/segsplit/var.log 2>&1
done
python scripts/seg_var.py longest >> gpurun_out/segsplit/reps.log 2>&1
EXSUM_LIB=paper_1505_05571_b200/lib/variants/segsplit.so python scripts/seg_var.py longest >> gpurun_out/segsplit/reps.log 2>&1
true
