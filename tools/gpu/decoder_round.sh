timeout 900 python -m pytest tests/test_gpu_decoder.py -x -q 2>&1 | tail -3 > gpurun_out/all.log
timeout 900 ncu --set full --clock-control none -k regex:"attn_(fwd|bwd)" -c 3 -o gpurun_out/attn_full -f python tools/decoder_step.py --layers 1 --steps 1 > gpurun_out/ncu_attn.log 2>&1
