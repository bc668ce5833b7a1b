mkdir -p gpurun_out/refresh
P=gpurun_out/refresh
timeout 600 python bench.py --config 4 --p2p --nccl --steps 10 --warmup 3 --no-cpu-baseline > $P/bench_c4_p2p_nccl.json 2> $P/bench_c4_p2p_nccl.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > $P/bench_torchrun1.json 2> $P/bench_torchrun1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --steps 10 --warmup 3 --impl reference > $P/ref_torchrun1.json 2> $P/ref_torchrun1.err
timeout 600 python bench.py --config 5 --steps 20 --warmup 5 > $P/bench_c5.json 2> $P/bench_c5.err
timeout 600 python bench.py --config 1 > $P/bench_c1.json 2> $P/bench_c1.err
timeout 600 python bench.py --config 1 --impl reference > $P/ref_c1.json 2> $P/ref_c1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"exsum_segment" -s 4 -c 4 -o $P/r02_c5b python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c5.csv python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $P/launch_c5.log 2>&1
true
