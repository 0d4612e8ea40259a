#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
: > gpurun_out/dbg.log
run() { echo "$* :: $(env "$@" timeout 120 python tools/run_blk.py --n $N --b $B --reps 1 2>&1 | tail -1 | cut -c1-100)" >> gpurun_out/dbg.log; }
N=9000 B=256 run SKL_MIN_CLUSTER_W=48
N=9000 B=256 run SKL_MIN_CLUSTER_W=40
N=16384 B=256 run SKL_MIN_CLUSTER_W=48
N=16384 B=256 run SKL_MIN_CLUSTER_W=32
SKL_MIN_CLUSTER_W=40 timeout 600 python -m pytest tests/test_gpu_blocked.py -x -q -m gpu -k "config3 or config2" >> gpurun_out/dbg.log 2>&1
for w in 64 56 48 40; do echo "w=$w $(SKL_MIN_CLUSTER_W=$w timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/dbg.log; done
