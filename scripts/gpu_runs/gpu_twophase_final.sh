# two-phase plain sums: full GPU suite, two-phase sweep, A/B vs one phase, bench lines, ncu of the windowed kernel
mkdir -p gpurun_out/tpf
P=gpurun_out/tpf
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $P/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
timeout 1500 python scripts/two_phase_sweep.py --cases 32 --seed 9 > $P/sweep.log 2>&1
timeout 1500 python scripts/ab_variants.py --cases c4,c3,c2 --rounds 4 default onephase > $P/time.log 2>&1
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $P/ref.json 2>&1
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $P/bench.json 2> $P/bench.err
timeout 600 python bench.py --config 4 --hold 5 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > $P/hold_c4.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exsum_wsum_kernel -s 3 -c 1 -o $P/r02_c4_wsum python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c4.csv python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c4.log 2>&1
true
