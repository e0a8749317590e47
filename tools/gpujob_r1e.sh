nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c4_default.json 2> gpurun_out/bench_c4_default.err; echo bench rc=$?; cat gpurun_out/bench_c4_default.json
