timeout 900 python -m pytest tests/test_gpu_abjoin.py -q -x > gpurun_out/gputests_ab.log 2>&1; echo ab tests rc=$?; tail -30 gpurun_out/gputests_ab.log | grep -E "passed|failed|Error|assert" | head -20
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gputests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4b.json 2> gpurun_out/bench_c4b.err; echo bench rc=$?; python -c "import json; d=json.load(open('gpurun_out/bench_c4b.json')); print(d['ms_per_step'], d['phases_ms'], d['e2e'])"
