timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1
MLORA_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --config c5 --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_c5_2.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1
