for r in 1 2; do
SKMP_JOIN_WARMUP=0 python tools/join_bench.py | sed "s/^/nowarm /"
python tools/join_bench.py | sed "s/^/warm   /"
SKMP_JOIN_WARMUP=0 python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/nowarm /"
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 | sed "s/^/warm   /"
done
timeout 900 python -m pytest tests/test_gpu_mp.py -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gputests.log
