set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
for r in 1 2; do for v in vnorthr cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py | sed "s/^/$v /"
done; done 2>&1 | grep -v "^+"
for v in vnorthr cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py --k 4 --n 2000000 --reps 2 | sed "s/^/$v /"
done 2>&1 | grep -v "^+"
timeout 900 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or abjoin or stream or detect or multirank or fullsize" > gpurun_out/r2_tests_rthr.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_tests_rthr.log
