# round 2: finalize (division-free, immediate-offset staging) + join ring-index spill fix; parity, A/B, C4 and C5 bench
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or abjoin or detect or stream or c3_full or c4_dynamic or experiment or dims or multirank" > gpurun_out/r2_tests4.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests4.log
for r in 1 2; do for v in qtlive cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py | sed "s/^/$v /"
done; done 2>&1 | tee gpurun_out/r2_qt_ab.txt
for f in smem reg; do SKMP_FIN_IMPL=$f timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_fin3_$f.json 2>/dev/null; echo "fin $f rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r2_c4_fin3_$f.json'));print('$f', d['ms_per_step'], d['phases_ms'], d['roofline']['pipe_frac'])"; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c5b.json 2> gpurun_out/r2_bench_c5b.err; echo c5 rc=$?; python -c "import json;d=json.load(open('gpurun_out/r2_bench_c5b.json'));print(d['value'], d['ms_per_step'], d['phases_ms'], d['roofline']['pipe_frac'], d['e2e']['value'])"
