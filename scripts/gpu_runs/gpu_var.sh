mkdir -p gpurun_out/var
for i in 1 2 3 4; do
  for o in longest index; do
    timeout 300 python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --seg-order $o 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 $o', d['roofline']['kernel_ms'], d['value'], d['clocks']['power_w_median'])" >> gpurun_out/var/var.log 2>&1
  done
  timeout 300 python bench.py --config 4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['roofline']['kernel_ms'], d['value'], d['clocks']['power_w_median'])" >> gpurun_out/var/var.log 2>&1
done
true
