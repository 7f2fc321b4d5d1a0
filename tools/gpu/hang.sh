timeout 600 python -m pytest tests/test_gpu_decoder.py tests/test_gpu_executor.py -x -q 2>&1 | tail -3 > gpurun_out/all.log
timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_decoder.py -x -q -k "rescale or attention_fwd_bwd" 2>&1 | tail -2 >> gpurun_out/all.log
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_decoder.py -x -q -k "rescale or attention_fwd_bwd or long" 2>&1 | tail -2 >> gpurun_out/all.log
timeout 600 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_decoder.py -x -q -k "attention_fwd_bwd" 2>&1 | tail -2 >> gpurun_out/all.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_" -c 5 --csv --log-file gpurun_out/attn_all.csv python tools/decoder_step.py --layers 1 --steps 1 > /dev/null 2>&1
timeout 600 python tools/decoder_probe.py --cfg chatglm2-6b --jobs 6 --seqs 4 --len 512 > gpurun_out/probe.log 2>&1
timeout 600 python tools/decoder_probe.py --cfg llama-7b --layers 4 --jobs 4 --seqs 4 --len 512 >> gpurun_out/probe.log 2>&1
