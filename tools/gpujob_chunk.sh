python tools/join_bench.py
python tools/join_bench.py --k 32 --n 100000 --m 128
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:join_x2_kernel -c 1 python tools/join_bench.py --reps 1 2>&1 | grep -E "dram__|gpu__time" 
timeout 900 python -m pytest tests/test_gpu_mp.py tests/test_gpu_abjoin.py -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gputests.log
