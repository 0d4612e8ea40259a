#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python tools/panel_sweep.py > gpurun_out/sweep.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_cluster -s 3 -c 1 -o gpurun_out/panel_c2 python tools/run_blk.py --reps 1 > gpurun_out/ncu_c2.log 2>&1
