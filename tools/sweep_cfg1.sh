#!/bin/bash
# config 1 (n=512 two-step through the blocked driver): panel width x rows per CTA
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/multi.log 2>&1; echo "rc=$?" >> gpurun_out/multi.log
: > gpurun_out/sweep_cfg1.log
for nb in 96 128 192 256 511; do for rows in 8 16 32 64; do
  echo "nb=$nb rows=$rows $(SKL_GPU_NB=$nb SKL_CLUSTER_ROWS=$rows SKL_MIN_CLUSTER_W=1 timeout 60 python tools/run_twostep.py 512 2>&1 | tail -1)" >> gpurun_out/sweep_cfg1.log
done; done
