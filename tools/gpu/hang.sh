timeout 1200 python tools/c4_executor.py > gpurun_out/c4_executor.jsonl 2> gpurun_out/c4_executor.err
C4_CFG=c3 timeout 1200 python tools/c4_executor.py > gpurun_out/c3_model.jsonl 2> gpurun_out/c3_model.err
