set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2m_c4.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:finalize_hw -s 3 -c 1 -o gpurun_out/r2m_finalize_c4 -f python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2m_ncu_fin.log 2>&1; echo ncu1 rc=$?
