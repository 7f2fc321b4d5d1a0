set -x
timeout 600 python -m pytest tests/test_gpu_decoder.py -x -q 2>&1 | tail -15 > gpurun_out/all.log
timeout 300 python tools/decoder_probe.py --cfg tiny-llama --jobs 2 --seqs 2 --len 64 --parity > gpurun_out/probe.log 2>&1
timeout 300 python tools/decoder_probe.py --cfg chatglm2-6b --layers 2 --jobs 6 --seqs 2 --len 256 --parity >> gpurun_out/probe.log 2>&1
timeout 600 python tools/decoder_probe.py --cfg chatglm2-6b --jobs 6 --seqs 4 --len 512 >> gpurun_out/probe.log 2>&1
timeout 600 python tools/decoder_probe.py --cfg llama-7b --layers 4 --jobs 4 --seqs 4 --len 512 >> gpurun_out/probe.log 2>&1
