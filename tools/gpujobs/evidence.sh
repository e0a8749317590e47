# round-1 final evidence: default bench, ncu launch list, ncu full capture of the join and finalize
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_c4_final.json 2> gpurun_out/bench_c4_final.err; echo bench rc=$?
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_x2_kernel -s 3 -c 1 -o gpurun_out/prof_join_final python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
