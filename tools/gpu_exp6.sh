cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
L=paper_2411_09859_b200/_lib
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_blocked.py tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/exp6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/exp6_tests.log
timeout 300 python tools/kernel_split.py 16384 256 > gpurun_out/exp6.log 2>&1
timeout 300 python tools/kernel_split.py 16384 256 >> gpurun_out/exp6.log 2>&1
SKEWLTL_B200_LIB=$L/libskewltl_b200_prof.so MULTI_NAMES=1 timeout 200 python tools/push_phases.py 16384:128 >> gpurun_out/exp6.log 2>&1
