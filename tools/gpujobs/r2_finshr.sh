# round 2: sub-warp finalize with the warp-shared row super-window (cur) vs per-group row buffers (vshr0)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or detect or abjoin or stream or fullsize or dims or multirank" > gpurun_out/r2_tests_finshr.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests_finshr.log
for v in vshr0 cur vshr0 cur; do
  L=""; if [ "$v" != cur ]; then L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_fin$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_c4_fin$v.json'));print('$v c4', round(d['ms_per_step'],2), {k: round(x,3) for k,x in d['phases_ms'].items()})"
done 2>&1 | grep -v "^+"
timeout 600 ncu --kernel-name regex:finalize --launch-count 1 --clock-control none --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2_finshr_ncu.txt 2>&1; echo ncu rc=$?; grep -E "gpu__time|inst_executed|issue|warps|registers|bank" gpurun_out/r2_finshr_ncu.txt | head -8
