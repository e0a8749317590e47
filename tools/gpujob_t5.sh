nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_mix tools/micro/pipe_mix.cu > /dev/null 2>&1 && /tmp/pipe_mix
timeout 600 python -m pytest tests/test_gpu_mp.py tests/test_gpu_experiment.py -q -x 2>&1 | tail -2
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
timeout 900 python tools/exp_synthetic.py --trials 10 > gpurun_out/exp41_t10.jsonl 2> gpurun_out/exp41.err; echo exp rc=$?; cat gpurun_out/exp41_t10.jsonl
