#!/bin/bash
for rt in 64 128 256 512; do
  SKL_CLUSTER_ROWS=$rt python tools/run_blk.py --reps 2 | sed "s/^/rows_target=$rt /"
done
