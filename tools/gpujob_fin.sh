timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gputests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4c.json 2> gpurun_out/bench_c4c.err; echo bench rc=$?; python -c "import json; d=json.load(open('gpurun_out/bench_c4c.json')); print(d['ms_per_step'], d['phases_ms'], d['e2e'])"
