# round 2 ncu: full capture of the join (C4 shape) and the finalize (C4 bench), launch list of the C5 bench
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
python tools/join_bench.py --reps 1 > gpurun_out/r2_jb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:join_x2 -c 1 -o gpurun_out/r2_join_x2_c4 -f python tools/join_bench.py --reps 1 > gpurun_out/r2_ncu_join.log 2>&1; echo ncu1 rc=$?
python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:finalize -s 3 -c 1 -o gpurun_out/r2_finalize_c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_fin.log 2>&1; echo ncu2 rc=$?
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c5_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_c5_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_c5.log 2>&1; echo ncu3 rc=$?
python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_plain2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches.csv python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_c4.log 2>&1; echo ncu4 rc=$?
