#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_solve.py tests/test_gpu_float32.py -x -q -m gpu > gpurun_out/solve_tests.log 2>&1; echo "rc=$?" >> gpurun_out/solve_tests.log
SKL_SOLVE_FUSED=0 timeout 600 python -m pytest tests/test_gpu_solve.py -x -q -m gpu > gpurun_out/solve_tests0.log 2>&1; echo "rc=$?" >> gpurun_out/solve_tests0.log
: > gpurun_out/solve_ab.log
for rep in 1 2; do for f in 0 1; do
  echo "fused=$f $(SKL_SOLVE_FUSED=$f timeout 300 python tools/run_solve.py 4096 2>&1 | tr '\n' ' ' | cut -c1-300)" >> gpurun_out/solve_ab.log
done; done
echo "fused=1 $(timeout 300 python tools/run_solve.py 16384 2>&1 | tr '\n' ' ' | cut -c1-300)" >> gpurun_out/solve_ab.log
