# round 2: finalize with prefetched statistics, faster window prep; parity + C4 A/B + FP64 join size sweep
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or abjoin or detect or stream or c3_full or c4_dynamic or experiment or sketch or dims" > gpurun_out/r2_tests3.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests3.log
for f in smem reg; do SKMP_FIN_IMPL=$f timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_fin2_$f.json 2>/dev/null; echo "fin $f rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r2_c4_fin2_$f.json'));print('$f', d['ms_per_step'], d['phases_ms'], d['roofline']['pipe_frac'])"; done
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 2
