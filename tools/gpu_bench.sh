#!/bin/bash
# bench line + batched ncu capture (round-1 refresh)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:batched -s 2 -c 1 -o gpurun_out/bt64_v2 python tools/run_batched.py f64 8192 > gpurun_out/ncu_bt.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:batched --csv python tools/run_batched.py f64 8192 > gpurun_out/bt_launch.csv 2>&1
