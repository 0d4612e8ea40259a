#!/bin/bash
# time config 2 / config 1 / (optionally config 3) under several environment settings
# usage: ENVS="A=1|A=2 B=3|" bash tools/gpu_envsweep.sh   ('|'-separated; empty = default)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/envsweep.log
IFS='|' read -ra CFGS <<< "$ENVS"
for rep in 1 2; do for c in "${CFGS[@]}"; do
  echo "[$c] $(env $c timeout 120 python tools/kernel_split.py 4096 128 2>&1 | tail -1)" >> gpurun_out/envsweep.log
  echo "[$c] $(env $c timeout 120 python tools/run_twostep.py 512 2>&1 | tail -1)" >> gpurun_out/envsweep.log
done; done
if [ -n "$C3" ]; then for c in "${CFGS[@]}"; do
  echo "[$c] $(env $c timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/envsweep.log
done; fi
