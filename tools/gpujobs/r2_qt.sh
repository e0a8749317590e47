# round 2: ring-row variants of the FP32 join (SKMP_X2_QT 0..3; cur = 2) + the async mp_create tests + full parity (top-K)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
for r in 1 2; do for v in qt0 qt1 qt3 cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py | sed "s/^/$v /"
done; done 2>&1 | grep -v "^+" | tee gpurun_out/r2_qtvar_ab.txt
for v in qt1 cur; do
  if [ "$v" = cur ]; then L=""; else L=$PWD/paper_2311_03393_b200/libsketchmp_$v.so; fi
  SKMP_LIB=$L python tools/join_bench.py --k 4 --n 2000000 --reps 2 | sed "s/^/$v /"
done 2>&1 | grep -v "^+" | tee -a gpurun_out/r2_qtvar_ab.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_tests5.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests5.log
timeout 900 python tools/full_parity.py --config c3 > gpurun_out/r2_full_parity_c3.json 2> gpurun_out/r2_fp_c3.err; echo fp3 rc=$?
timeout 1200 python tools/full_parity.py --config c4 > gpurun_out/r2_full_parity_c4.json 2> gpurun_out/r2_fp_c4.err; echo fp4 rc=$?
cat gpurun_out/r2_full_parity_c3.json gpurun_out/r2_full_parity_c4.json
