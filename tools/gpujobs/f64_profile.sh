# ncu --set full of the FP64 join at the C2 shape (k=16, n=20000, m=100)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:join_kernel -c 1 -o gpurun_out/prof_join_f64_c2b python tools/join_bench.py --k 16 --n 20000 --m 100 --dtype f64 --reps 1 > gpurun_out/ncu_f64.log 2>&1; echo ncu rc=$?
