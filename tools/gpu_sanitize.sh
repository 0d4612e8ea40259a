#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the small-n workload
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/sanitize
CS=compute-sanitizer
run() {  # name, env, tool, extra
  local name=$1 envs=$2 tool=$3; shift 3
  env $envs timeout 1500 $CS --tool $tool "$@" --print-limit 50 python tools/sanitize_cases.py 300 \
     > gpurun_out/sanitize/${name}_${tool}.log 2>&1
  echo "$name $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE_CASES_OK' gpurun_out/sanitize/${name}_${tool}.log | tr '\n' ' ')" >> gpurun_out/sanitize/summary.txt
}
: > gpurun_out/sanitize/summary.txt
run lean "SKL_PANEL_V2=1" memcheck
run lean "SKL_PANEL_V2=1" synccheck
run lean "SKL_PANEL_V2=1" racecheck --racecheck-report all
run oldpanel "SKL_PANEL_V2=0" memcheck
run oldpanel "SKL_PANEL_V2=0" racecheck --racecheck-report all
run multi "SKL_FORCE_MULTI=1" memcheck
run multi "SKL_FORCE_MULTI=1" racecheck --racecheck-report all
