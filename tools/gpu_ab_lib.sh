#!/bin/bash
# A/B of two builds of the library (AB_LIB_OLD vs the default build) on one box, parity tests first
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
OLD=${AB_LIB_OLD:-paper_2411_09859_b200/_lib/libskewltl_b200_vprev.so}
NEW=paper_2411_09859_b200/_lib/libskewltl_b200.so
timeout 900 python -m pytest tests/test_gpu_blocked.py tests/test_gpu_multi.py tests/test_gpu_twostep.py tests/test_gpu_unpivoted.py tests/test_gpu_float32.py tests/test_trace.py tests/test_gpu_solve.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
: > gpurun_out/ab.log
for rep in 1 2; do for L in $OLD $NEW; do
  echo "$(basename $L) $(SKEWLTL_B200_LIB=$L timeout 120 python tools/kernel_split.py 4096 128 2>&1 | tail -1)" >> gpurun_out/ab.log
  echo "$(basename $L) $(SKEWLTL_B200_LIB=$L timeout 120 python tools/run_twostep.py 512 2>&1 | tail -1)" >> gpurun_out/ab.log
done; done
for L in $OLD $NEW; do
  echo "$(basename $L) $(SKEWLTL_B200_LIB=$L timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/ab.log
done
for L in $OLD $NEW; do
  echo "$(basename $L) $(SKEWLTL_B200_LIB=$L timeout 300 python tools/time_batched.py 2>&1 | tail -2 | tr '\n' ' ')" >> gpurun_out/ab.log
done
timeout 600 python -m pytest tests/test_gpu_batched.py -x -q -m gpu > gpurun_out/ab_tests_b.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests_b.log
SKEWLTL_B200_LIB=$OLD timeout 300 python tools/bitcmp.py /tmp/bc_old.npz
SKEWLTL_B200_LIB=$NEW timeout 300 python tools/bitcmp.py /tmp/bc_new.npz
python tools/bitcmp.py /tmp/bc_old.npz /tmp/bc_new.npz >> gpurun_out/ab.log 2>&1
