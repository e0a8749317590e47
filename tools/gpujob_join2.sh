# gpu tests (scalar default + x2 parity on the mp tests), then join timings of the variants
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/gputests.log
SKMP_JOIN_IMPL=x2 timeout 600 python -m pytest tests/test_gpu_mp.py tests/test_gpu_fullsize.py -q -x > gpurun_out/gputests_x2.log 2>&1; echo x2 tests rc=$?; tail -5 gpurun_out/gputests_x2.log
python tools/join_bench.py
SKMP_JOIN_IMPL=x2 python tools/join_bench.py | sed 's/^/x2mb1 /'
for mb in 12 16; do SKMP_JOIN_IMPL=x2 SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_x2mb$mb.so python tools/join_bench.py | sed "s/^/x2mb$mb /"; done
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
