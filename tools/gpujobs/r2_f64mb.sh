# round 2: FP64 join occupancy caps (launch bounds 18 / 20 CTAs per SM: 96 registers) vs 16 (114 registers)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
for r in 1 2; do for v in mb18 mb20 cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 2 | sed "s/^/$v /"
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/$v /"
done; done 2>&1 | grep -v "^+"
for v in mb18 mb20 cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py --k 16 --n 2000000 --m 100 --dtype f64 --reps 1 | sed "s/^/$v /"
done 2>&1 | grep -v "^+"
