#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
L=paper_2411_09859_b200/_lib
for v in "$@"; do
  echo "== lib$v" >> gpurun_out/bt_time.log
  SKEWLTL_B200_LIB=$L/libskewltl_b200$v.so timeout 300 python tools/time_batched.py >> gpurun_out/bt_time.log 2>&1
done
