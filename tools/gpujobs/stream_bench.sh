#!/bin/bash
# f4 streaming latency at the C4 train size -> gpurun_out/stream_bench.jsonl
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python tools/stream_bench.py > gpurun_out/stream_bench.jsonl 2> gpurun_out/stream_bench.err
echo "rc=$?"; cat gpurun_out/stream_bench.jsonl
