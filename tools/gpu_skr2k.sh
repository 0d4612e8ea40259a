#!/bin/bash
# skr2k microbench: parity tests, A/B timing of the prologue, per-launch durations, one full ncu capture of the GEMM
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/skr2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/skr2k_tests.log
timeout 300 python tools/run_skr2k.py 30 > gpurun_out/skr2k.log 2>&1
SKL_SKR2K_PREP=0 timeout 300 python tools/run_skr2k.py 30 >> gpurun_out/skr2k.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/run_skr2k.py > gpurun_out/skr2k_launches.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_lower -s 2 -c 1 -o gpurun_out/skr2k_gemm python tools/run_skr2k.py > gpurun_out/ncu_skr2k.log 2>&1
