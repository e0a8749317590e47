# round-1 evidence: gpu tests, bench (C4), ncu launch list + full capture of the join, §4.1 experiment
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench rc=$?; cat gpurun_out/bench_c4.json
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:join_x2_kernel -s 3 -c 1 -o gpurun_out/prof_join_c4 python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
timeout 900 python tools/exp_synthetic.py --trials 100 > gpurun_out/exp41_t100.jsonl 2> gpurun_out/exp41.err; echo exp rc=$?; cat gpurun_out/exp41_t100.jsonl
