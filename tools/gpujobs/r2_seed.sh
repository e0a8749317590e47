# round 2: seed change (FP32 x2 + FP64) + re-seed interval A/B (16384 vs 32768) at C4 and C5-length
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or detect or abjoin or stream or dims or c3_full or multirank or fullsize" > gpurun_out/r2_tests_seed.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests_seed.log
for r in 1 2; do for L in 0 32768; do
  python tools/join_bench.py --reseed $L | sed "s/^/L=$L /"
done; done 2>&1 | grep -v "^+" | tee gpurun_out/r2_seed_ab.txt
for L in 0 32768; do python tools/join_bench.py --k 4 --n 2000000 --reps 2 --reseed $L | sed "s/^/L=$L /"; done 2>&1 | grep -v "^+" | tee -a gpurun_out/r2_seed_ab.txt
python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 2 | tee -a gpurun_out/r2_seed_ab.txt
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | tee -a gpurun_out/r2_seed_ab.txt
