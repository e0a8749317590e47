python tools/join_bench.py
SKMP_JOIN_IMPL=x2 python tools/join_bench.py | sed 's/^/x2 /'
SKMP_JOIN_IMPL=x2 timeout 600 python -m pytest tests/test_gpu_mp.py -q -x 2>&1 | tail -2
