#!/bin/bash
# one in-situ ncu capture of the config-2 cluster panel (4th panel launch), with source
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_cluster -s 3 -c 1 -o gpurun_out/panel_c2 -f python tools/run_blk.py --reps 1 > gpurun_out/ncu_panel.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_panel.log
