timeout 900 python -m pytest tests/test_gpu_decoder.py -x -q 2>&1 | tail -3 > gpurun_out/all.log
MLORA_ATTN_HSPLIT=4 timeout 900 python -m pytest tests/test_gpu_decoder.py -x -q -k "attention" 2>&1 | tail -3 >> gpurun_out/all.log
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_decoder.py -x -q -k "attention_fwd_bwd" 2>&1 | tail -3 >> gpurun_out/all.log
