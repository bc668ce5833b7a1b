mkdir -p gpurun_out/segflat
P=gpurun_out/segflat
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exsum_segflat_kernel -s 1 -c 1 -o $P/flat_c5_v4 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_flat4.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/segclaim.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:exsum_segmented_kernel -s 1 -c 1 -o $P/claim_c5 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --seg-mode claim > $P/ncu_claim.log 2>&1
true
