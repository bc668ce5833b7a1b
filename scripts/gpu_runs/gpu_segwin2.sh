mkdir -p gpurun_out/segwin
for i in 1 2; do
python scripts/seg_var.py longest >> gpurun_out/segwin/var2.log 2>&1
EXSUM_LIB=paper_1505_05571_b200/lib/variants/segwin4.so python scripts/seg_var.py longest >> gpurun_out/segwin/var2.log 2>&1
EXSUM_LIB=paper_1505_05571_b200/lib/variants/segwin1.so python scripts/seg_var.py longest >> gpurun_out/segwin/var2.log 2>&1
EXSUM_LIB=paper_1505_05571_b200/lib/variants/segwin16.so python scripts/seg_var.py longest >> gpurun_out/segwin/var2.log 2>&1
python scripts/seg_var.py index >> gpurun_out/segwin/var2.log 2>&1
done
true
