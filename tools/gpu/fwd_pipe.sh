# attention forward (software-pipelined tcgen05): parity first, then the launch list
timeout 300 python -m pytest tests/test_gpu_decoder.py -x -q > gpurun_out/fwdp_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/fwdp_tests.log
for i in 1 2 3; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_fwd" -c 2 --csv --log-file gpurun_out/fwdp_$i.csv python tools/decoder_step.py --layers 1 --steps 2 > /dev/null 2>&1
done
tail -3 gpurun_out/fwdp_tests.log
