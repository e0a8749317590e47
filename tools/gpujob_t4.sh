timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/gputests.log
SKMP_JOIN_IMPL=scalar timeout 600 python -m pytest tests/test_gpu_mp.py tests/test_gpu_fullsize.py -q -x > gpurun_out/gputests_scalar.log 2>&1; echo scalar tests rc=$?; tail -3 gpurun_out/gputests_scalar.log
python tools/join_bench.py
SKMP_JOIN_IMPL=scalar python tools/join_bench.py | sed 's/^/scalar /'
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_d64x4.so python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed 's/^/d64x4 /'
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_d64x4.so timeout 600 python -m pytest tests/test_gpu_mp.py -q -x -k f64 2>&1 | tail -2
