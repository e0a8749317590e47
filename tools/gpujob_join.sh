# usage: bash tools/gpujob_join.sh [pytest-args]   (build, gpu tests, join timings)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
if [ "${SKIP_TESTS:-0}" != 1 ]; then
timeout 900 python -m pytest tests -m gpu -q -x ${@} > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/gputests.log
fi
python tools/join_bench.py
SKMP_JOIN_IMPL=x2 python tools/join_bench.py
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
