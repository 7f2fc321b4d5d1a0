timeout 900 python -m pytest tests/test_gpu_decoder.py tests/test_gpu_executor.py tests/test_gpu_model.py -x -q 2>&1 | tail -15 > gpurun_out/all.log
