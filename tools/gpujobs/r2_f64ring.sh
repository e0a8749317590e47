set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -k "test_gpu_mp or detect or abjoin or stream or dims or dist1 or comm or multirank or c_abi or sketch or experiment" > gpurun_out/r2_tests_f64r.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_tests_f64r.log
python tools/join_bench.py --k 16 --n 200000 --m 100 --dtype f64 --reps 2
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
python tools/join_bench.py --k 4 --n 2000 --m 50 --dtype f64
