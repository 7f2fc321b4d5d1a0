# dK/dV cluster head split sweep on the warp-specialised kernel (launch-list times)
for hs in 1 2 4 8; do
MLORA_ATTN_HSPLIT=$hs timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_bwd_dkv" -c 2 --csv --log-file gpurun_out/hs_$hs.csv python tools/decoder_step.py --layers 1 --steps 2 > /dev/null 2>&1
done
