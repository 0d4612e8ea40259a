#!/bin/bash
# round-2 evidence: phase tables (single + multi-cluster), ncu --set full of one multi-cluster panel launch and
# one single-cluster launch, config-3 launch list
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
L=paper_2411_09859_b200/_lib
SKEWLTL_B200_LIB=$L/libskewltl_b200_prof.so timeout 200 python tools/push_phases.py 512:96 2048:96 4096:96 > gpurun_out/ev_push_phases.log 2>&1
SKEWLTL_B200_LIB=$L/libskewltl_b200_prof.so MULTI_NAMES=1 timeout 200 python tools/push_phases.py 16384:128 > gpurun_out/ev_multi2_phases.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_multi2 -s 2 -c 1 -o gpurun_out/ev_multi2 -f python tools/run_blk.py --n 16384 --b 256 --reps 0 > gpurun_out/ev_ncu_multi2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_push -s 4 -c 1 -o gpurun_out/ev_push -f python tools/run_blk.py --reps 0 > gpurun_out/ev_ncu_push.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_n16384.csv python tools/run_blk.py --n 16384 --b 256 --reps 0 > gpurun_out/ev_ncu_l3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_launches_n4096.csv python tools/run_blk.py --reps 0 > gpurun_out/ev_ncu_l2.log 2>&1
