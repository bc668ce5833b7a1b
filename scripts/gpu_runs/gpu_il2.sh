mkdir -p gpurun_out/il2
for i in 1 2 3; do TV_OVERLAP=1 TV_CONFIGS=2,3,4,6 python scripts/time_variants.py ranges pf0 pf2 backoff15 >> gpurun_out/il2/time.log 2>&1; done
true
