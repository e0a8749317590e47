# AB-join timings (f1): C4-like (train n = 200k, test 100k, k = 64, m = 256, FP32) and C2-like FP64
python tools/join_bench.py --ab 100000
python tools/join_bench.py --ab 200000
python tools/join_bench.py --k 16 --n 12000 --ab 8000 --m 100 --dtype f64
