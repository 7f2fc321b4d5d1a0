timeout 300 python -m pytest tests/test_gpu_decoder.py -x -q 2>&1 | tail -2 > gpurun_out/all.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_rope" -c 2 --csv --log-file gpurun_out/rope.csv python tools/decoder_step.py --layers 1 --steps 1 > /dev/null 2>&1
