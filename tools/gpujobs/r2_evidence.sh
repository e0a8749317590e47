# round 2 evidence: full GPU suite + smoke, the driver's bench lines (reference arm, C5 default, C4), join ncu capture
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2j_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2j_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo smoke rc=$?; cat gpurun_out/r2j_smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2j_bench_reference.json 2> gpurun_out/r2j_ref.err; echo ref rc=$?
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2j_bench_c5.json 2> gpurun_out/r2j_c5.err; echo c5 rc=$?; cat gpurun_out/r2j_bench_c5.json
timeout 900 python bench.py --config c4 --steps 20 --warmup 5 > gpurun_out/r2j_bench_c4.json 2> gpurun_out/r2j_c4.err; echo c4 rc=$?
python tools/join_bench.py --reps 1 > gpurun_out/r2j_jb.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:join_x2 -c 1 -o gpurun_out/r2j_join_x2_c4 -f python tools/join_bench.py --reps 1 > gpurun_out/r2j_ncu_join.log 2>&1; echo ncu rc=$?
