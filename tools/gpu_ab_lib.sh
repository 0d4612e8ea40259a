#!/bin/bash
# A/B two builds of the library on one box: LIBS="a.so|b.so" bash tools/gpu_ab_lib.sh  (C3=1 adds config 3)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
L=paper_2411_09859_b200/_lib
: > gpurun_out/ab_lib.log
IFS='|' read -ra LS <<< "$LIBS"
for rep in 1 2; do for l in "${LS[@]}"; do
  echo "[$l] $(SKEWLTL_B200_LIB=$L/$l timeout 120 python tools/kernel_split.py 4096 128 2>&1 | tail -1)" >> gpurun_out/ab_lib.log
  echo "[$l] $(SKEWLTL_B200_LIB=$L/$l timeout 120 python tools/kernel_split.py 512 128 2>&1 | tail -1)" >> gpurun_out/ab_lib.log
done; done
if [ -n "$C3" ]; then for l in "${LS[@]}"; do
  echo "[$l] $(SKEWLTL_B200_LIB=$L/$l timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/ab_lib.log
done; fi
