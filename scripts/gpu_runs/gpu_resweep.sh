# knob re-sweep with the robust protocol (scripts/ab_variants.py: idle pauses, variants interleaved)
mkdir -p gpurun_out/resweep
P=gpurun_out/resweep
timeout 1500 python scripts/ab_variants.py --cases c4,c3 --rounds 3 default pf0 pf2 ldg1 ldg0 ldg4 w8s65 w9v8 nofast backoff15 il0 v6 v7 xorimad cta132 > $P/sum_knobs.log 2>&1
timeout 900 python scripts/ab_variants.py --cases c5 --rounds 3 default seg6 seg7 segtail2 segtail8 pf2 pf0 > $P/seg_knobs.log 2>&1
true
