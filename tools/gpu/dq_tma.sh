# dQ with Q / dO by TMA: parity, then the launch list
timeout 300 python -m pytest tests/test_gpu_decoder.py tests/test_gpu_executor.py -x -q > gpurun_out/dq_tests.log 2>&1; echo "exit $?" >> gpurun_out/dq_tests.log
for i in 1 2; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_bwd" -c 4 --csv --log-file gpurun_out/dq_$i.csv python tools/decoder_step.py --layers 1 --steps 2 > /dev/null 2>&1
done
tail -2 gpurun_out/dq_tests.log
