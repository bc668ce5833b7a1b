mkdir -p gpurun_out
(for v in c1_p0 c2_p0 c2_p128 c2_p512 c4_p0 c4_p128; do echo "== $v"; taskset -c 2 ./scripts/probes/host_kernel_$v 50000000; done) > gpurun_out/r2b_host_kernel.log 2>&1
(cd scripts/probes && ./small_bench) > gpurun_out/r2b_small_bench.log 2>&1
python scripts/e2e_probe.py > gpurun_out/r2b_e2e_probe.log 2>&1
timeout 900 python -m pytest tests/test_p2p_procs.py tests/test_context_gpu.py tests/test_synth.py -m gpu -q --timeout 600 > gpurun_out/r2b_gpu_tests.log 2>&1
true
