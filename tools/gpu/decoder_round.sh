timeout 900 python -m pytest tests/test_gpu_executor.py tests/test_gpu_parity.py -x -q 2>&1 | tail -15 > gpurun_out/all.log
timeout 600 python tools/c3_executor.py > gpurun_out/c3.jsonl 2>&1
