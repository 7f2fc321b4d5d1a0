for i in 1 2 3; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_fwd" -c 2 --csv --log-file gpurun_out/fwd_tc_$i.csv python tools/decoder_step.py --layers 1 --steps 2 > /dev/null 2>&1
MLORA_ATTN_TC=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_fwd" -c 2 --csv --log-file gpurun_out/fwd_mma_$i.csv python tools/decoder_step.py --layers 1 --steps 2 > /dev/null 2>&1
done
timeout 600 python tools/decoder_probe.py --cfg chatglm2-6b --jobs 6 --seqs 4 --len 512 > gpurun_out/probe.log 2>&1
