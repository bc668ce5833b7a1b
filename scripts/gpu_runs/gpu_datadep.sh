mkdir -p gpurun_out/datadep
P=gpurun_out/datadep
timeout 600 python scripts/data_dep.py > $P/dd2.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/sumfix1.so timeout 600 python scripts/data_dep.py >> $P/dd2.log 2>&1
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/sumfix2.so timeout 600 python scripts/data_dep.py >> $P/dd2.log 2>&1
true
