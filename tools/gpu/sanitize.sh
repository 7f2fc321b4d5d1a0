for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_decoder.py -x -q -k "attention_fwd_bwd or swiglu_and_norm or deterministic" > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_summary.log
done
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -x -q -k "fuse or fuzz and (0 or 1)" > gpurun_out/san_fuse.log 2>&1; echo "fuse memcheck rc=$?" >> gpurun_out/san_summary.log
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_model.py -x -q > gpurun_out/san_ce.log 2>&1; echo "ce memcheck rc=$?" >> gpurun_out/san_summary.log
