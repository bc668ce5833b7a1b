# round 2, fourth session: final evidence on the ripple build (default)
mkdir -p gpurun_out/final8
P=gpurun_out/final8
python scripts/build_variants.py debug > $P/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/ref.json 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench.json 2> $P/bench.err
for c in 2 3 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $P/bench_c$c.json 2> $P/bench_c$c.err; done
for c in 2 3 4 5; do timeout 600 python bench.py --config $c --hold 5 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > $P/hold_c$c.json 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exsum_wsum_kernel -s 3 -c 1 -o $P/r02_c4_final python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exsum_sum_kernel -s 3 -c 1 -o $P/r02_c2_final python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c2.log 2>&1
for c in 3 4 5; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c$c.csv python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c$c.log 2>&1; done
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/debug.so timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests_debug.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/debug.so timeout 600 python scripts/sanitize_run.py > $P/sanitize_debug.log 2>&1
timeout 500 python scripts/long_sweep.py --seconds 300 --seed 21 > $P/long_sweep.log 2>&1
timeout 1200 python scripts/two_phase_sweep.py --cases 16 --seed 5 > $P/tp_sweep.log 2>&1
true
