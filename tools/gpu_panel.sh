#!/bin/bash
# panel change: parity tests of the blocked driver + config 2/3 kernel split
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blocked.py tests/test_gpu_unpivoted.py tests/test_gpu_dist.py -x -q > gpurun_out/pt.log 2>&1; echo "rc=$?" >> gpurun_out/pt.log
timeout 300 python tools/kernel_split.py 4096 128 > gpurun_out/psplit.log 2>&1
timeout 300 python tools/kernel_split.py 16384 256 >> gpurun_out/psplit.log 2>&1
