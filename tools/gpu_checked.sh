#!/bin/bash
# compute-sanitizer is closed on this GPU pool: run the GPU suite against the checked build
# (device asserts on the panel's exchange invariants and indices; -DSKL_CHECKED)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SKEWLTL_B200_LIB=paper_2411_09859_b200/_lib/libskewltl_b200_vchecked.so timeout 1800 python -m pytest tests -m gpu -q \
  --deselect tests/test_gpu_cfg5.py::test_config5_golden > gpurun_out/checked_tests.log 2>&1
echo "rc=$?" >> gpurun_out/checked_tests.log
