# longer randomized sweeps on the final (ripple) build, with the two carry-chain distributions
mkdir -p gpurun_out/sweep2
P=gpurun_out/sweep2
timeout 800 python scripts/long_sweep.py --seconds 600 --seed 31 > $P/long_sweep_a.log 2>&1
timeout 800 python scripts/long_sweep.py --seconds 600 --seed 32 > $P/long_sweep_b.log 2>&1
true
