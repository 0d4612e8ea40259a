#!/bin/bash
# A/B of an environment knob: OLD env (AB_ENV_OLD, e.g. SKL_PANEL_V2=0) vs default; parity subset first
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blocked.py tests/test_gpu_twostep.py tests/test_gpu_push.py tests/test_gpu_unpivoted.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
: > gpurun_out/ab.log
for rep in 1 2 3; do
  echo "old $(env $AB_ENV_OLD timeout 120 python tools/kernel_split.py 4096 128 2>&1 | tail -1)" >> gpurun_out/ab.log
  echo "new $(timeout 120 python tools/kernel_split.py 4096 128 2>&1 | tail -1)" >> gpurun_out/ab.log
  echo "old $(env $AB_ENV_OLD timeout 120 python tools/run_twostep.py 512 2>&1 | tail -1)" >> gpurun_out/ab.log
  echo "new $(timeout 120 python tools/run_twostep.py 512 2>&1 | tail -1)" >> gpurun_out/ab.log
done
echo "old $(env $AB_ENV_OLD timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/ab.log
echo "new $(timeout 300 python tools/kernel_split.py 16384 256 2>&1 | tail -1)" >> gpurun_out/ab.log
timeout 600 python tools/panel_sweep.py --ns 512,4096 --widths 16,32,64,96 >> gpurun_out/ab.log 2>&1
