# occupancy experiment: 16-slot window (config 4's exponent range), 8/12/16 warps per SM (timing only)
mkdir -p gpurun_out/window
P=gpurun_out/window
timeout 1500 python scripts/ab_variants.py --cases c4 --rounds 3 default win16v4 win16v3 win20v3 win24v2 win32v2 win16v4s8 > $P/time2.log 2>&1
true
