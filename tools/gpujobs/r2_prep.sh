# round 2: where the C4 mp_prep phase's time goes (r2k bench: 12.6 ms vs 1.7 ms in r2j)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
python tools/phase_probe.py 2>&1 | tail -12
for v in hw reg hw; do
  F=""; if [ "$v" = reg ]; then F=reg; fi
  SKMP_FIN_IMPL=$F timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_prep_$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_prep_$v.json'));print('$v c4', round(d['ms_per_step'],2), {k: round(x,3) for k,x in d['phases_ms'].items()})"
done 2>&1 | grep -v "^+"
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x -k full_bench > gpurun_out/r2_multirank_e2e.log 2>&1; echo mr rc=$?; tail -30 gpurun_out/r2_multirank_e2e.log
