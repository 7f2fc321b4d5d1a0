# compute-sanitizer over the r02 kernel changes: the narrowed shared-input and grouped
# forward down-projections (tests/test_gpu_down_multi.py: NB 2..5, several tiles per CTA
# pair, rank groups 1..4, empty jobs, K tails) and the base GEMM's LoRA k-step skipping
# (forward / backward parity on ragged layouts, the C2 layer step).
rm -f gpurun_out/san_r02_summary.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_gpu_down_multi.py -x -q > gpurun_out/san_r02_dm_$tool.log 2>&1
  echo "down_multi $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_r02_dm_$tool.log | tr '\n' ' ')" >> gpurun_out/san_r02_summary.log
done
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -x -q -k "forward_backward_parity or layer_step or fuzz" > gpurun_out/san_r02_parity.log 2>&1
echo "parity memcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_r02_parity.log | tr '\n' ' ')" >> gpurun_out/san_r02_summary.log
# the cluster masked-CE row pass (bulk copies, st.async partial exchange)
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python -m pytest tests/test_gpu_model.py -x -q -k masked_ce > gpurun_out/san_r02_ce_$tool.log 2>&1
  echo "masked_ce $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/san_r02_ce_$tool.log | tr '\n' ' ')" >> gpurun_out/san_r02_summary.log
done
