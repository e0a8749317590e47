python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
python tools/join_bench.py --k 4 --n 2000 --m 50 --dtype f64
python tools/join_bench.py
python tools/join_bench.py --k 32 --n 100000 --m 128
timeout 900 python -m pytest tests/test_gpu_mp.py tests/test_gpu_abjoin.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gputests.log
