cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
L=paper_2411_09859_b200/_lib
for d in f64 f32; do
SKEWLTL_B200_LIB=$L/libskewltl_b200_vbprof.so timeout 120 python tools/batched_prof.py $d 8192 $([ $d = f64 ] && echo 28 || echo 19) >> gpurun_out/bt_time.log 2>&1
done
SKEWLTL_B200_LIB=$L/libskewltl_b200_vbprof.so timeout 120 python tools/batched_prof.py f64 296 1 >> gpurun_out/bt_time.log 2>&1
