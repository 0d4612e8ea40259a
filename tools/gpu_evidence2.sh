#!/bin/bash
# ncu of one multi-cluster panel launch.  The cooperative multi-cluster kernel spins on L2 flags
# between clusters: kernel replay (memory restore) and SASS-patching sections (SourceCounters)
# break it ("illegal instruction"), so: application replay, hardware-counter sections only.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 ncu --replay-mode application --clock-control none --section LaunchStats --section SpeedOfLight --section WarpStateStats --section SchedulerStats --section MemoryWorkloadAnalysis --section Occupancy --section ComputeWorkloadAnalysis -k regex:panel_multi2 -s 2 -c 1 -o gpurun_out/ev_multi2 -f python tools/run_blk.py --n 16384 --b 256 --reps 0 > gpurun_out/ev_ncu_multi2.log 2>&1
timeout 900 ncu --replay-mode application --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_n16384.csv python tools/run_blk.py --n 16384 --b 256 --reps 0 > gpurun_out/ev_ncu_l3.log 2>&1
