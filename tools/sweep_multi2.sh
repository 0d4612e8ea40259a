#!/bin/bash
# config-3 plan sweep after the push-mode panel: multi-cluster width cap x cluster count
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/sweep_multi2.log
for w in 96 128 160 192; do
  echo "SKL_MULTI_NB=$w $(SKL_MULTI_NB=$w timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/sweep_multi2.log
done
for q in 6 8; do
  echo "SKL_MULTI_Q=$q $(SKL_MULTI_Q=$q timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/sweep_multi2.log
done
