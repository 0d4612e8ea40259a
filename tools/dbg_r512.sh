#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/dbg.log
run() { echo "$* :: $(env "$@" timeout 120 python tools/run_blk.py --n $N --b $B --reps 1 2>&1 | tail -1 | cut -c1-120)" >> gpurun_out/dbg.log; }
N=8193 B=256 run SKL_MIN_CLUSTER_W=48
N=9000 B=128 run SKL_MIN_CLUSTER_W=48
N=9000 B=96 run SKL_MIN_CLUSTER_W=48
N=9000 B=256 run SKL_MIN_CLUSTER_W=48 SKL_GPU_NB=48
N=9000 B=256 run SKL_MIN_CLUSTER_W=48 SKL_MULTI_NB=96
N=9000 B=256 run SKL_MIN_CLUSTER_W=56
N=8700 B=256 run SKL_MIN_CLUSTER_W=48
