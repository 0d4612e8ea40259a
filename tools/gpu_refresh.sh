#!/bin/bash
# bench line + config-2 launch list + panel DRAM bytes + one full panel capture (round-1 refresh)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
[ -n "$WITH_BENCH" ] && { timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; }
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_blk.py --reps 1 > gpurun_out/launches_c2.csv 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:panel_cluster --csv python tools/run_blk.py --reps 1 > gpurun_out/panel_dram.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_cluster -s 3 -c 1 -o gpurun_out/panel_c2 -f python tools/run_blk.py --reps 1 > gpurun_out/ncu_panel.log 2>&1
