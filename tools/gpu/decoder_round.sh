timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_decoder.py -x -q 2>&1 | tail -3 > gpurun_out/all.log
