# Round-2 evidence: bench lines (configs 2-5 + reference arms), ncu --set full of the
# dominant kernels, serialized launch lists.  Outputs under gpurun_out/prof2/.
mkdir -p gpurun_out/prof2
P=gpurun_out/prof2
for c in 4 2 3 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $P/bench_c$c.json 2> $P/bench_c$c.err; done
for c in 4 5; do timeout 600 python bench.py --impl reference --config $c --steps 20 --warmup 5 > $P/bench_ref_c$c.json 2>&1; done
python scripts/e2e_probe.py --threads 16,15 --reps 8 > $P/e2e_probe.log 2>&1
for c in 4 2 3; do timeout 600 ncu --set full --clock-control none --import-source on -k regex:exsum_sum_kernel -s 3 -c 1 -o $P/r02_c$c python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c$c.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"exsum_segment" -s 3 -c 4 -o $P/r02_c5 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c5.log 2>&1
for c in 4 5; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c$c.csv python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c$c.log 2>&1; done
ls -la $P
