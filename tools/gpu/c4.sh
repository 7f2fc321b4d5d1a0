timeout 1500 python tools/c4_executor.py > gpurun_out/c4_executor.jsonl 2> gpurun_out/c4_executor.err
