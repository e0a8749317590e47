# round 2: join x2 chunk staging by cp.async.bulk (TMA 1-D bulk copies + mbarrier, SKMP_X2_BULK) vs per-lane cp.async
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_bulk.so timeout 900 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or abjoin or stream or detect or multirank" > gpurun_out/r2_tests_bulk.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_tests_bulk.log
for r in 1 2; do for v in cur bulk; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py | sed "s/^/$v /"
  SKMP_LIB=$L python tools/join_bench.py --k 4 --n 2000000 --reps 2 | sed "s/^/$v c5len /"
done; done 2>&1 | grep -v "^+"
