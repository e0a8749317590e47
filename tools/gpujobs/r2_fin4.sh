set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or stream or abjoin" > gpurun_out/r2_tests7.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_tests7.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_fin5.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_c4_fin5.json'));print(d['ms_per_step'], d['phases_ms'], d['roofline']['pipe_frac'])"
python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c4_launches_b.csv python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
