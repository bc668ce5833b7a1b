mkdir -p gpurun_out/segwin
timeout 600 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py -m gpu -q -k "segment or config5 or seg" --timeout 500 > gpurun_out/segwin/tests.log 2>&1
for i in 1 2 3; do
  for v in default segwin1 segwin4 segwin16; do
    if [ $v = default ]; then L=""; else L="EXSUM_LIB=paper_1505_05571_b200/lib/variants/$v.so"; fi
    env $L timeout 300 python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['roofline']['kernel_ms'], d['value'])" >> gpurun_out/segwin/var.log 2>&1
  done
  timeout 300 python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --seg-order index 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('index', d['roofline']['kernel_ms'], d['value'])" >> gpurun_out/segwin/var.log 2>&1
done
true
