#!/bin/bash
# staged cross-cluster exchange: parity (forced multi at small n, config 3 golden) + A/B timing
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/stage_multi.log 2>&1; timeout 900 python -m pytest tests/test_gpu_blocked.py -x -q -m gpu > gpurun_out/stage_tests.log 2>&1; echo "rc=$?" >> gpurun_out/stage_tests.log
for st in 0 1; do
  SKL_MULTI_STAGE=$st timeout 300 python tools/kernel_split.py 16384 256 > gpurun_out/stage_split_$st.log 2>&1
  SKL_MULTI_STAGE=$st timeout 300 python tools/kernel_split.py 8192 256 >> gpurun_out/stage_split_$st.log 2>&1
done
SKEWLTL_B200_LIB=paper_2411_09859_b200/_lib/libskewltl_b200_prof.so timeout 200 python tools/cluster_prof.py 16384 256 > gpurun_out/cprof_stage.log 2>&1
