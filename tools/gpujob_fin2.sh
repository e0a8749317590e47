nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_rate tools/micro/fp64_rate.cu > /dev/null 2>&1 && /tmp/fp64_rate
timeout 900 python -m pytest tests/test_gpu_mp.py tests/test_gpu_detect.py tests/test_gpu_abjoin.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gputests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4d.json 2> gpurun_out/bench_c4d.err; echo bench rc=$?; python -c "import json; d=json.load(open('gpurun_out/bench_c4d.json')); print(d['ms_per_step'], d['phases_ms'])"
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4d.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:finalize_kernel -s 1 -c 1 -o gpurun_out/prof_fin_c4 python bench.py $ARGS > gpurun_out/ncu_fin.log 2>&1; echo ncu2 rc=$?
