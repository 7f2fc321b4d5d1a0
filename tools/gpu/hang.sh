timeout 600 python -m pytest tests/test_gpu_decoder.py tests/test_gpu_executor.py -x -q 2>&1 | tail -8 > gpurun_out/all.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_" -c 6 --csv --log-file gpurun_out/attn_all.csv python tools/decoder_step.py --layers 1 --steps 1 > /dev/null 2>&1
timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_decoder.py -x -q -k "rescale or attention_fwd_bwd" 2>&1 | tail -2 >> gpurun_out/all.log
