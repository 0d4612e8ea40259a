cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/full_tests.log 2>&1; echo "rc=$?" >> gpurun_out/full_tests.log
ENVS="SKL_FINAL_ROWS=0|SKL_FINAL_ROWS=600|SKL_FINAL_ROWS=600 SKL_GPU_NB=128" bash tools/gpu_envsweep.sh
