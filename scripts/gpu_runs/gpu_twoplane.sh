# two sign planes in the windowed pass (EXSUM_W_PLANES=2): tests, sweep, A/B vs one plane, bench, ncu
mkdir -p gpurun_out/tpl
P=gpurun_out/tpl
python scripts/build_variants.py oneplane > $P/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x --timeout 900 -k "two_phase or config or golden" > $P/tests_sel.log 2>&1
timeout 1200 python scripts/two_phase_sweep.py --cases 32 --seed 12 > $P/sweep.log 2>&1
timeout 1200 python scripts/ab_variants.py --cases c4,c3,c2 --rounds 4 default oneplane > $P/time.log 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-e2e > $P/bench.json 2> $P/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exsum_wsum_kernel -s 3 -c 1 -o $P/r02_c4_w2 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c4.csv python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c4.log 2>&1
true
