# round 2 last check after the FP64 small-grid instance: full GPU suite + smoke
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2w_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2w_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2w_smoke.log 2>&1; echo smoke rc=$?; cat gpurun_out/r2w_smoke.log
