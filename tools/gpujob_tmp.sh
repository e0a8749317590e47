python tools/join_bench.py
python tools/join_bench.py --dtype f64 --k 16 --n 20000 --m 100
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
