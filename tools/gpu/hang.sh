timeout 600 python -m pytest tests/test_gpu_decoder.py tests/test_gpu_model.py -x -q 2>&1 | tail -2 > gpurun_out/all.log
MLORA_BENCH_LAYERS=2 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/b.log 2>&1
