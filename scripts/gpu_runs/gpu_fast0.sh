# ripple + per-vector vote: vectors of normal terms skip the e = 0 handling and the Inf/NaN watch (EXSUM_RIPPLE_FAST0)
mkdir -p gpurun_out/fast0
P=gpurun_out/fast0
python scripts/build_variants.py rfast0 > $P/build.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c3,c5,n01,c2 --rounds 3 default rfast0 > $P/time.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/rfast0.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > $P/tests.log 2>&1
for c in 3 5; do EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/rfast0.so timeout 600 python bench.py --config $c --hold 5 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > $P/hold_c$c.json 2>&1; done
for c in 3 5; do timeout 600 python bench.py --config $c --hold 5 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > $P/hold_default_c$c.json 2>&1; done
true
