python tools/join_bench.py --dtype f64 --k 16 --n 20000 --m 100 | sed "s/^/c2 /"
python tools/join_bench.py --dtype f32 --k 16 --n 20000 --m 100 | sed "s/^/c2f32 /"
python tools/join_bench.py --dtype f64 --k 4 --n 2000 --m 50 | sed "s/^/c1 /"
python tools/join_bench.py --dtype f32 --k 32 --n 100000 --m 128 | sed "s/^/c3 /"
python tools/join_bench.py
