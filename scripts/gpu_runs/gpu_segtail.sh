mkdir -p gpurun_out/segtail
timeout 900 python -m pytest tests/test_gpu.py tests/test_sweep_gpu.py -m gpu -q -x --timeout 600 -k "seg or config5" > gpurun_out/segtail/tests.log 2>&1
for i in 1 2 3; do
  python scripts/seg_var.py longest >> gpurun_out/segtail/reps.log 2>&1
  for v in segtail0 segtail16 segtailall; do
    EXSUM_LIB=paper_1505_05571_b200/lib/variants/$v.so python scripts/seg_var.py longest >> gpurun_out/segtail/reps.log 2>&1
  done
  python scripts/seg_var.py index >> gpurun_out/segtail/reps.log 2>&1
done
true
