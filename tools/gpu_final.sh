#!/bin/bash
# round-end style check: full GPU suite, smoke, bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final_bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/final_ref.log
