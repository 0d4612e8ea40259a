#!/bin/bash
# in-situ ncu captures of the config-2 lean panel (5th launch: 16 CTAs x ~230 rows), with source
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_push -s 4 -c 1 -o gpurun_out/push_c2 -f python tools/run_blk.py --reps 1 > gpurun_out/ncu_push.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_push.log
