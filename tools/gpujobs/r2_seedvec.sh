# round 2: float4 seed loads; parity + join timings + C5 bench
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or abjoin or stream or detect or fullsize or multirank or experiment" > gpurun_out/r2_tests_sv.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests_sv.log
for r in 1 2; do python tools/join_bench.py; done
python tools/join_bench.py --k 4 --n 2000000 --reps 2
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench_c5_sv.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_bench_c5_sv.json'));print(d['value'], d['ms_per_step'], d['phases_ms'], d['roofline']['pipe_frac'])"
# f1 AB-join and f4 streaming with the round-2 kernels, the §4.1 experiment re-run
python tools/join_bench.py --ab 100000 | tee gpurun_out/r2_abjoin.txt
python tools/join_bench.py --ab 200000 | tee -a gpurun_out/r2_abjoin.txt
timeout 600 python tools/stream_bench.py > gpurun_out/r2_stream_bench.jsonl 2> /dev/null; echo stream rc=$?
timeout 1200 python tools/exp_synthetic.py --trials 100 > gpurun_out/r2_exp41_t100.jsonl 2> gpurun_out/r2_exp41.err; echo exp rc=$?; cat gpurun_out/r2_exp41_t100.jsonl | cut -c1-300
