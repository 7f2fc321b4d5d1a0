set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mlora|adam|rowsq|loss_guard|reduce_splits" -s 44 -c 22 -o gpurun_out/bench_step_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn|ce_rows|swiglu|rmsnorm|embed" -c 20 -o gpurun_out/decoder_full -f python tools/decoder_step.py --layers 1 --steps 1 > gpurun_out/ncu_dec.log 2>&1
