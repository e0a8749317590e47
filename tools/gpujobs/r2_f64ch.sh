# round 2: FP64 join per-cell tests in 4 independent predicate chains (cur) vs one serial chain (ch1)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
for r in 1 2; do for v in ch1 cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 2 | sed "s/^/$v /"
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/$v /"
done; done 2>&1 | grep -v "^+"
for v in ch1 cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 2000000 --m 100 --dtype f64 --reps 1 | sed "s/^/$v /"
done 2>&1 | grep -v "^+"
timeout 900 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or abjoin or multirank or detect or dims or stream" > gpurun_out/r2_tests_f64ch.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests_f64ch.log
timeout 600 ncu --kernel-name regex:join_kernel --launch-skip 1 --launch-count 1 --clock-control none --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 1 > gpurun_out/r2_f64ch_ncu.txt 2>&1; echo ncu rc=$?; grep -E "gpu__time|pipe|issue|warps|registers" gpurun_out/r2_f64ch_ncu.txt
