timeout 900 python -m pytest tests/test_gpu_sketch.py -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/gputests.log | grep -E "passed|failed|Error|assert" 
