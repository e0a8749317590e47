# round 2: FP64 join high-word filters (rows: f64row; rows + columns: cur) vs the round-1 kernel (f64old)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or detect or abjoin or stream or dims or dist1 or comm or multirank or c_abi or sketch" > gpurun_out/r2_tests_f64.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests_f64.log
for r in 1 2; do for v in f64old f64row cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/$v /"
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 2 | sed "s/^/$v /"
done; done 2>&1 | grep -v "^+" | tee gpurun_out/r2_f64_ab.txt
python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:join_kernel -c 1 -o gpurun_out/r2_join_f64 -f python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 1 > gpurun_out/r2_ncu_f64.log 2>&1; echo ncu rc=$?
