# round 2 final kernels: every profile row of C3, C4 (dynamic pipeline) and two whole C5 series vs tier B, top-K vs the oracle
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
timeout 2400 python tools/full_parity.py --config c3 > gpurun_out/r2u_parity_c3.json 2> gpurun_out/r2u_parity_c3.err; echo c3 rc=$?; cat gpurun_out/r2u_parity_c3.json
timeout 2400 python tools/full_parity.py --config c4 > gpurun_out/r2u_parity_c4.json 2> gpurun_out/r2u_parity_c4.err; echo c4 rc=$?; cat gpurun_out/r2u_parity_c4.json
timeout 2400 python tools/c5_tierb.py > gpurun_out/r2u_c5_tierb.json 2> gpurun_out/r2u_c5_tierb.err; echo c5 rc=$?; cat gpurun_out/r2u_c5_tierb.json
