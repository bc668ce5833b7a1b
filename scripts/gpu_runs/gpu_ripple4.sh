# ripple (default build): second knob sweep + held lines
mkdir -p gpurun_out/ripple4
P=gpurun_out/ripple4
python scripts/build_variants.py noripple rv4 rv5 rv7 rseg5 rseg6 rseg8 rsegahead rnosplit > $P/build.log 2>&1
timeout 2400 python scripts/ab_variants.py --cases c3,c5,c2 --rounds 3 default noripple rv4 rv5 rv7 rseg5 rseg6 rseg8 rsegahead rnosplit > $P/time.log 2>&1
for c in 3 5; do timeout 600 python bench.py --config $c --hold 5 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > $P/hold_c$c.json 2>&1; done
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/noripple.so timeout 600 python bench.py --config 3 --hold 5 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > $P/hold_c3_noripple.json 2>&1
true
