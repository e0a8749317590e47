timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -s --durations=5 > gpurun_out/fullsize.log 2>&1; echo rc=$?; tail -15 gpurun_out/fullsize.log
