# round 2: finalize ranks FP32 candidate sets in FP32 (SKMP_FIN_SEL32) vs all-FP64 (sel64)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or detect or abjoin or stream or dims or c3_full or c4_dynamic or c5_end or experiment" > gpurun_out/r2_tests_sel32.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests_sel32.log; grep -E "ties|top-" gpurun_out/r2_tests_sel32.log | head
for v in sel64 cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_c4_$v.json'));print('$v', d['ms_per_step'], d['phases_ms'])"
done
python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:finalize --csv --log-file gpurun_out/r2_fin_sel32.csv python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
timeout 900 python tools/full_parity.py --config c3 > gpurun_out/r2_fp_c3_sel32.json 2>/dev/null; cat gpurun_out/r2_fp_c3_sel32.json
