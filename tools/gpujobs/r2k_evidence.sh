# round 2 evidence after the sub-warp finalize: full GPU suite + smoke, the driver's bench lines
# (reference arm, C5 default, C4), launch lists (C4, C5) and an ncu --set full of the finalize
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2k_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2k_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo smoke rc=$?; cat gpurun_out/r2k_smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2k_bench_reference.json 2> gpurun_out/r2k_ref.err; echo ref rc=$?
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2k_bench_c5.json 2> gpurun_out/r2k_c5.err; echo c5 rc=$?; cat gpurun_out/r2k_bench_c5.json
timeout 900 python bench.py --config c4 --steps 20 --warmup 5 > gpurun_out/r2k_bench_c4.json 2> gpurun_out/r2k_c4.err; echo c4 rc=$?
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2k_c4_launches.csv python bench.py --config c4 $ARGS > gpurun_out/r2k_ncu_c4.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2k_c5_launches.csv python bench.py $ARGS > gpurun_out/r2k_ncu_c5.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:finalize -s 3 -c 1 -o gpurun_out/r2k_finalize_c4 -f python bench.py --config c4 $ARGS > gpurun_out/r2k_ncu_fin.log 2>&1; echo ncu3 rc=$?
