mkdir -p gpurun_out
(for v in c1_p0 c1_p512 c1_p1024 c2_p0 c2_p256 c2_p512 c2_p1024 c2_p2048; do echo "== $v"; taskset -c 2 ./scripts/probes/host_kernel_$v 50000000 | grep 50000000; ./scripts/probes/host_kernel_$v 1000000000 15; done) > gpurun_out/r2c_host_kernel.log 2>&1
true
