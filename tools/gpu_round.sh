#!/bin/bash
# One GPU call: gpu tests, kernel split at config 2/3, bench line.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests.log
timeout 300 python tools/kernel_split.py 4096 128 > gpurun_out/split.log 2>&1
timeout 300 python tools/kernel_split.py 16384 256 >> gpurun_out/split.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
