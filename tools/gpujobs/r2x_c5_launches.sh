# round 2: C5 launch list with the final kernels (only libsketchmp's kernels profiled: the device-side
# input generation's torch kernels run unprofiled)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py $ARGS > gpurun_out/r2x_c5_plain.json 2>/dev/null; echo plain rc=$?
timeout 1500 ncu --kernel-name-base demangled -k regex:skmp:: --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2x_c5_launches.csv python bench.py $ARGS > gpurun_out/r2x_ncu_c5.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/r2x_ncu_c5.log
