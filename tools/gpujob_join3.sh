timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/gputests.log
python tools/join_bench.py
SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_pubinl.so python tools/join_bench.py | sed 's/^/pubinl /'
for v in x2mb16 pubinl_x2mb12 pubinl_x2mb16; do SKMP_JOIN_IMPL=x2 SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_$v.so python tools/join_bench.py | sed "s/^/$v /"; done
SKMP_JOIN_IMPL=x2 SKMP_LIB=$PWD/paper_2311_03393_b200/libsketchmp_x2mb16.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_x2_kernel -c 1 -o gpurun_out/joinx2_mb16 python tools/join_bench.py --reps 1 > gpurun_out/ncu_x2mb16.log 2>&1; echo ncu rc=$?
