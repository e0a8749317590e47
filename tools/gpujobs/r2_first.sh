# round 2, first GPU pass: build, the new / changed GPU tests, smoke, the C5 default bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
free -g; nproc
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -k "grid_stride or multirank or dims or dist1 or c_abi or stream or c5_end or comm or detect" > gpurun_out/r2_tests1.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/r2_tests1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo bench rc=$?; cat gpurun_out/r2_bench_c5.json; tail -5 gpurun_out/r2_bench_c5.err
