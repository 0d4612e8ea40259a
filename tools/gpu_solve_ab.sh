#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_solve.py tests/test_gpu_float32.py -x -q -m gpu > gpurun_out/solve_tests.log 2>&1; echo "rc=$?" >> gpurun_out/solve_tests.log
: > gpurun_out/solve_ab.log
for rep in 1 2; do for L in paper_2411_09859_b200/_lib/libskewltl_b200_vprev.so paper_2411_09859_b200/_lib/libskewltl_b200.so; do
  echo "$(basename $L) $(SKEWLTL_B200_LIB=$L timeout 300 python tools/run_solve.py 4096 2>&1 | tr '\n' ' ' | cut -c1-300)" >> gpurun_out/solve_ab.log
done; done
echo "new $(timeout 300 python tools/run_solve.py 16384 2>&1 | tr '\n' ' ' | cut -c1-300)" >> gpurun_out/solve_ab.log
