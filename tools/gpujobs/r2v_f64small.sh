# round 2: FP64 join small-grid instance (96 registers, 18 warps/SM) for grids <= 16 waves
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
for r in 1 2; do
  python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/cur /"
  python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 2 | sed "s/^/cur /"
  python tools/join_bench.py --k 4 --n 2000 --m 50 --dtype f64 | sed "s/^/cur c1 /"
done 2>&1 | grep -v "^+"
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2v_c2.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2v_c2.json'));print('c2', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['phases_ms'].items()})"
timeout 1200 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or abjoin or detect or dims or stream or multirank" > gpurun_out/r2v_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2v_tests.log
