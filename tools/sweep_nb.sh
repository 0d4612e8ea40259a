#!/bin/bash
for nb in 48 64 80 96 0; do
  SKL_GPU_NB=$nb python tools/run_blk.py --reps 2 | sed "s/^/gpu_nb=$nb /"
done
