timeout 900 ncu --set full --clock-control none -k regex:"attn_(fwd_tc|bwd_dq_ws|bwd_dkv_ws)" -c 3 -o gpurun_out/attn_tc_full -f python tools/decoder_step.py --layers 1 --steps 1 > /dev/null 2>&1
