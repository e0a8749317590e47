# every row of C3 and C4 against tier B (one-off evidence; ~10 min on a 16-core host)
free -g | head -2
timeout 2400 python tools/full_parity.py --config c3 > gpurun_out/full_parity_c3.json 2> gpurun_out/full_parity_c3.err; echo c3 rc=$?; cat gpurun_out/full_parity_c3.json; tail -2 gpurun_out/full_parity_c3.err
timeout 2400 python tools/full_parity.py --config c4 > gpurun_out/full_parity_c4.json 2> gpurun_out/full_parity_c4.err; echo c4 rc=$?; cat gpurun_out/full_parity_c4.json; tail -2 gpurun_out/full_parity_c4.err
