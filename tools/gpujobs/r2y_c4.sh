# round 2: C4 bench line again (the r2k line's mean held one outlier step)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build.log; exit 1; }
for r in 1 2; do
timeout 900 python bench.py --config c4 --steps 20 --warmup 5 > gpurun_out/r2y_bench_c4_$r.json 2> gpurun_out/r2y_c4_$r.err; echo c4 rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2y_bench_c4_$r.json'));print('c4', round(d['ms_per_step'],2), d['value'], d['roofline']['pipe_frac'], d['e2e']['value'], {k: round(x,3) for k,x in d['phases_ms'].items()})"
done
