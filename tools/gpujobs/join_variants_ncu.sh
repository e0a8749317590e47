# build, gpu tests, join timings, then one ncu --set full capture of each FP32 join variant
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
if [ "${SKIP_TESTS:-0}" != 1 ]; then
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/gputests.log
fi
python tools/join_bench.py
SKMP_JOIN_IMPL=x2 python tools/join_bench.py
python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64
TAG=${TAG:-cur}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_kernel -c 1 -o gpurun_out/join_${TAG} python tools/join_bench.py --reps 1 > gpurun_out/ncu_join_${TAG}.log 2>&1; echo ncu1 rc=$?
SKMP_JOIN_IMPL=x2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_x2_kernel -c 1 -o gpurun_out/joinx2_${TAG} python tools/join_bench.py --reps 1 > gpurun_out/ncu_joinx2_${TAG}.log 2>&1; echo ncu2 rc=$?
