#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/bt.log 2>&1; echo "rc=$?" >> gpurun_out/bt.log
bash tools/gpu_batched.sh "$@"
