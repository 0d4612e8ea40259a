#!/bin/bash
# quick A/B of two library builds (AB_LIB_OLD vs the default build): parity subset, then
# alternating kernel_split timings at config 2 / config 1 / config 3
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
OLD=${AB_LIB_OLD:-paper_2411_09859_b200/_lib/libskewltl_b200_vprev.so}
NEW=paper_2411_09859_b200/_lib/libskewltl_b200.so
timeout 900 python -m pytest tests/test_gpu_blocked.py tests/test_gpu_multi.py tests/test_gpu_twostep.py tests/test_gpu_push.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
: > gpurun_out/ab.log
for rep in 1 2 3; do for L in $OLD $NEW; do
  echo "$(basename $L) $(SKEWLTL_B200_LIB=$L timeout 120 python tools/kernel_split.py 4096 128 2>&1 | tail -1)" >> gpurun_out/ab.log
  echo "$(basename $L) $(SKEWLTL_B200_LIB=$L timeout 120 python tools/run_twostep.py 512 2>&1 | tail -1)" >> gpurun_out/ab.log
done; done
for L in $OLD $NEW; do
  echo "$(basename $L) $(SKEWLTL_B200_LIB=$L timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/ab.log
done
