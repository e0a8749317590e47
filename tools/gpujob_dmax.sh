python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
python tools/join_bench.py --k 4 --n 2000 --m 50 --dtype f64
timeout 900 python -m pytest tests/test_gpu_mp.py tests/test_gpu_detect.py tests/test_gpu_abjoin.py -m gpu -q -x -k "f64 or c1 or c2 or small" > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gputests.log
