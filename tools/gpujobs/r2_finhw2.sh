# round 2: half-warp finalize, register cap 128 (cur) vs 96 (vmb5), vs the full-warp kernel (reg)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
for v in reg cur vmb5 reg cur vmb5; do
  L=""; unset SKMP_FIN_IMPL
  if [ "$v" = reg ]; then export SKMP_FIN_IMPL=reg; elif [ "$v" != cur ]; then L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_c4_fin$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/r2_c4_fin$v.json'));print('$v c4', round(d['ms_per_step'],2), {k: round(x,3) for k,x in d['phases_ms'].items()})"
done 2>&1 | grep -v "^+"
unset SKMP_FIN_IMPL
timeout 900 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or detect or abjoin or stream or fullsize" > gpurun_out/r2_tests_finhw2.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests_finhw2.log
for v in cur vmb5; do
  L=""; if [ "$v" != cur ]; then L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L timeout 600 ncu --kernel-name regex:finalize --launch-count 1 --clock-control none --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2_finhw2_ncu_$v.txt 2>&1; echo ncu $v rc=$?; grep -E "gpu__time|inst_executed|issue|warps|registers|bank" gpurun_out/r2_finhw2_ncu_$v.txt | head -8
done
