# a subset of GPU tests: bash tools/gpujobs/quick_tests.sh "<pytest -k expression>"
timeout 1200 python -m pytest tests -m gpu -q -x -k "$1" > gpurun_out/gputests_quick.log 2>&1; echo tests rc=$?; tail -15 gpurun_out/gputests_quick.log | grep -E "passed|failed|Error|assert" | head
