#!/bin/bash
# round-style check: full GPU suite, smoke, bench line, ncu launch list of one config-2 factorization
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full_tests.log 2>&1; echo "rc=$?" >> gpurun_out/full_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/full_smoke.log
timeout 900 python bench.py > gpurun_out/full_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/full_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'panel|gemm|pack|finalize|finish|compose' --csv --log-file gpurun_out/full_launches.csv python tools/run_blk.py --reps 1 > gpurun_out/full_ncu.log 2>&1
