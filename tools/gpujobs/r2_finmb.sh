# round 2: finalize register cap A/B (SKMP_FIN_MINB 1 / 5 / 6)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
for v in cur fmb5 fmb6; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_c4_$v.json'));print('$v', d['ms_per_step'], d['phases_ms'])"
done
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_fmb6.so timeout 900 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or detect or abjoin or stream" > gpurun_out/r2_tests_fmb6.log 2>&1; echo tests6 rc=$?; tail -2 gpurun_out/r2_tests_fmb6.log
