#!/bin/bash
# plan sweeps after the push-mode panel: config-2 GPU panel width, config-3 single-cluster width floor
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/sweep_push.log
for nb in 80 96 112 128; do
  echo "SKL_GPU_NB=$nb $(SKL_GPU_NB=$nb timeout 120 python tools/kernel_split.py 4096 128 2>&1 | tail -1)" >> gpurun_out/sweep_push.log
done
for w in 64 48 40 32; do
  echo "SKL_MIN_CLUSTER_W=$w $(SKL_MIN_CLUSTER_W=$w timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/sweep_push.log
done
for nb in 64 80 112; do
  echo "SKL_GPU_NB=$nb $(SKL_GPU_NB=$nb timeout 60 python tools/run_twostep.py 512 2>&1 | tail -1)" >> gpurun_out/sweep_push.log
done
