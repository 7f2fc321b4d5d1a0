set -x
timeout 900 python -m pytest tests/test_gpu_decoder.py tests/test_gpu_executor.py -x -q 2>&1 | tail -15 > gpurun_out/all.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv python tools/decoder_step.py --steps 2 > gpurun_out/dec_ncu.log 2>&1
timeout 600 python tools/decoder_probe.py --cfg chatglm2-6b --jobs 6 --seqs 4 --len 512 > gpurun_out/probe.log 2>&1
timeout 600 python tools/decoder_probe.py --cfg llama-7b --layers 4 --jobs 4 --seqs 4 --len 512 >> gpurun_out/probe.log 2>&1
