# final evidence of a round: default bench (C4, e2e pipelined, cpu_baseline), reference arm, C5 line,
# ncu launch list (time + DRAM bytes), ncu --set full of the join
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_c4_final.json 2> gpurun_out/bench_c4_final.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref rc=$?
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5 rc=$?
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_x2_kernel -s 3 -c 1 -o gpurun_out/prof_join_final python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
