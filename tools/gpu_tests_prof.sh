#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/full_tests.log 2>&1; echo "rc=$?" >> gpurun_out/full_tests.log
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:panel_push --csv --log-file gpurun_out/r02_panel_dram_n4096.csv python tools/run_blk.py --reps 1 > gpurun_out/ncu_dram.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_push -s 46 -c 1 -o gpurun_out/r02_panel_push_c2 python tools/run_blk.py --reps 1 > gpurun_out/ncu_full.log 2>&1
