timeout 600 python -m pytest tests/test_gpu_decoder.py -x -q 2>&1 | tail -2 > gpurun_out/all.log
for i in 1 2; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_fwd" -c 2 --csv --log-file gpurun_out/fwd_tc_$i.csv python tools/decoder_step.py --layers 1 --steps 2 > /dev/null 2>&1
done
