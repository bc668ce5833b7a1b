mkdir -p gpurun_out/misc
python scripts/latency_probe.py > gpurun_out/misc/latency.log 2>&1
TV_OVERLAP=1 TV_SUSTAIN=5 TV_CONFIGS=4,3 python scripts/time_variants.py > gpurun_out/misc/sustained.log 2>&1
true
