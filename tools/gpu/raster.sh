for rep in 1 2; do
for r in default 2 4 6 10 16 32; do
  if [ $r = default ]; then timeout 300 python tools/raster_probe.py 300; else MLORA_RASTER=$r timeout 300 python tools/raster_probe.py 300; fi
done
done > gpurun_out/raster.log 2>&1
