# two-phase plain sums (EXSUM_TWO_PHASE): tests, A/B against the one-phase build, bench line, launch list
mkdir -p gpurun_out/tp
P=gpurun_out/tp
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > $P/tests_all.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c4,c3 --rounds 4 default onephase > $P/time.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench.json 2> $P/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c4.csv python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c4.log 2>&1
true
