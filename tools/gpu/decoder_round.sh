timeout 900 python -m pytest tests/test_gpu_edge.py -x -q 2>&1 | tail -15 > gpurun_out/all.log
