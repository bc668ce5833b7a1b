# load-kind knob re-checked on the ripple / two-plane build (the kernels are L1-data-pipe bound now)
mkdir -p gpurun_out/ldg
P=gpurun_out/ldg
python scripts/build_variants.py ldg0 ldg1 ldg3 ldg4 > $P/build.log 2>&1
timeout 2400 python scripts/ab_variants.py --cases c4,c5,c3,c2 --rounds 3 default ldg0 ldg1 ldg3 ldg4 > $P/time.log 2>&1
true
