# ncu launch metrics of one C2 step's 14 base GEMMs for two builds (A/B)
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum
MLORA_LIBRARY=$PWD/paper_2312_02515_b200/libmlora_prev.so timeout 600 ncu --metrics $M --clock-control none -k regex:base_pair -s 14 -c 14 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ab_prev.csv 2>/dev/null
timeout 600 ncu --metrics $M --clock-control none -k regex:base_pair -s 14 -c 14 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ab_new.csv 2>/dev/null
