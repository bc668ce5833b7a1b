mkdir -p gpurun_out/segahead
EXSUM_LIB=$PWD/paper_1505_05571_b200/lib/variants/segahead.so timeout 900 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py tests/test_context_gpu.py -m gpu -q -x --timeout 600 -k "seg or config5" > gpurun_out/segahead/tests.log 2>&1
for i in 1 2 3; do
  python scripts/seg_var.py longest >> gpurun_out/segahead/reps.log 2>&1
  EXSUM_LIB=paper_1505_05571_b200/lib/variants/segahead.so python scripts/seg_var.py longest >> gpurun_out/segahead/reps.log 2>&1
done
true
