# round 2: finalize (FULL windows, 3-round argmin, explicit pass only for dd < 1) + qt3 join
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or abjoin or detect or stream or c3_full or c4_dynamic or dims or experiment or multirank" > gpurun_out/r2_tests6.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests6.log
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_fin4.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_c4_fin4.json'));print(d['ms_per_step'], d['phases_ms'], d['roofline']['pipe_frac'])"
python tools/join_bench.py --k 4 --n 2000000 --reps 2
python tools/join_bench.py
