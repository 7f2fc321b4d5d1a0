timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1
