cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
./tools/probes/fp64_lat > gpurun_out/fp64_lat.log 2>&1
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_formats.py tests/test_gpu_blocked.py -m gpu -q -x > gpurun_out/t3.log 2>&1; echo "rc=$?" >> gpurun_out/t3.log
timeout 300 python bench.py --steps 3 --warmup 3 --skip-other > gpurun_out/bench_quick.log 2>&1
