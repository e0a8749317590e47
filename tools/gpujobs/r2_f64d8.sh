# round 2: FP64 join D = 8 diagonals per thread (d8; 185 registers) and stale column-threshold
# registers after a publish (xr0) vs D = 4 with refreshed thresholds (cur)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
for r in 1 2; do for v in d8 xr0 cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 2 | sed "s/^/$v /"
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/$v /"
done; done 2>&1 | grep -v "^+"
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_d8.so timeout 900 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or abjoin or multirank or detect" > gpurun_out/r2_tests_f64d8.log 2>&1; echo tests d8 rc=$?; tail -3 gpurun_out/r2_tests_f64d8.log
