for r in 1 2; do
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_base.so python tools/join_bench.py | sed "s/^/base /"
python tools/join_bench.py | sed "s/^/new  /"
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_base.so python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/base /"
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/new  /"
done
SKMP_JOIN_IMPL=scalar SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_base.so python tools/join_bench.py | sed "s/^/base scalar /"
SKMP_JOIN_IMPL=scalar python tools/join_bench.py | sed "s/^/new  scalar /"
timeout 900 python -m pytest tests/test_gpu_mp.py tests/test_gpu_abjoin.py tests/test_gpu_detect.py -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gputests.log
