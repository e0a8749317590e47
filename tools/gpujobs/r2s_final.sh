# round 2 final check: full GPU suite + smoke (now with the FP32 join leg), the driver's default
# bench command and the reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2s_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2s_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1; echo smoke rc=$?; cat gpurun_out/r2s_smoke.log
timeout 1200 python bench.py > gpurun_out/r2s_bench_default.json 2> gpurun_out/r2s_bench_default.err; echo bench rc=$?; cat gpurun_out/r2s_bench_default.json
timeout 900 python bench.py --impl reference > gpurun_out/r2s_bench_reference.json 2> gpurun_out/r2s_ref.err; echo ref rc=$?; cat gpurun_out/r2s_bench_reference.json
