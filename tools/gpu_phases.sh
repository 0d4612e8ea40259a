#!/bin/bash
# panel phase clocks (profiling build) + one ncu --set full capture of a multi-cluster panel launch
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SKEWLTL_B200_LIB=paper_2411_09859_b200/_lib/libskewltl_b200_prof.so timeout 300 python tools/panel_phases.py 512:96 4096:96 16384:128 16384:32 --json gpurun_out/phases.json > gpurun_out/phases.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_cluster -s 1 -c 1 -o gpurun_out/panel_multi python tools/panel_phases.py 16384:128 > gpurun_out/ncu_multi.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_cluster -s 1 -c 1 -o gpurun_out/panel_single python tools/panel_phases.py 4096:96 > gpurun_out/ncu_single.log 2>&1
