timeout 300 python -m pytest tests/test_gpu_decoder.py -x -q 2>&1 | tail -15 > gpurun_out/all.log
for p in 1 0; do
MLORA_ATTN_PERS=$p timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_bwd_dq" -c 1 --csv --log-file gpurun_out/dq_p$p.csv python tools/decoder_step.py --layers 1 --steps 1 > /dev/null 2>&1
done
