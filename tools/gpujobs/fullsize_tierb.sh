nproc
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -s > gpurun_out/gputests_full.log 2>&1; echo tests rc=$?; grep -E "tier B|passed|failed|Error|assert" gpurun_out/gputests_full.log | head -10
