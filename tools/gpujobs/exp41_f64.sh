# the §4.1 experiment with FP64 joins (exact and sketched), fewer trials: is the success-rate
# finding an FP32 artefact?
timeout 2400 python tools/exp_synthetic.py --dtype f64 --trials 20 --d 250,1000,5000,10000 > gpurun_out/exp41_f64.jsonl 2> gpurun_out/exp41_f64.err; echo rc=$?; cat gpurun_out/exp41_f64.jsonl
