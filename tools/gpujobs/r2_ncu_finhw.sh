set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2l_c4.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:finalize_hw -s 3 -c 1 -o gpurun_out/r2l_finalize_c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2l_ncu_fin.log 2>&1; echo ncu1 rc=$?
python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 1 > gpurun_out/r2l_f64.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:join_kernel -c 1 -o gpurun_out/r2l_join_f64 -f python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 1 > gpurun_out/r2l_ncu_f64.log 2>&1; echo ncu2 rc=$?
