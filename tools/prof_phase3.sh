cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SKEWLTL_B200_LIB=paper_2411_09859_b200/_lib/libskewltl_b200_prof.so timeout 200 python tools/cluster_prof.py 4096 128 > gpurun_out/p3.log 2>&1
SKEWLTL_B200_LIB=paper_2411_09859_b200/_lib/libskewltl_b200_prof.so timeout 200 python tools/cluster_prof.py 16384 256 >> gpurun_out/p3.log 2>&1
