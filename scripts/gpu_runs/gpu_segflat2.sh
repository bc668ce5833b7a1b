mkdir -p gpurun_out/segflat
P=gpurun_out/segflat
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c5.csv python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c5.log 2>&1
true
