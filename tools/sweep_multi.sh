#!/bin/bash
# config-3 panel plan sweep: co-resident clusters (SKL_MULTI_Q) x panel width cap (SKL_MULTI_NB)
N=${N:-16384}; B=${B:-256}; DIST=${DIST:-uniform}
for q in ${QS:-4 6 9}; do for w in ${WS:-96 128 192 256}; do
  r=$(SKL_MULTI_Q=$q SKL_MULTI_NB=$w timeout 120 python tools/run_cfg5.py --n $N --b $B --dist $DIST --reps 2 --no-check 2>/dev/null | tail -1)
  echo "Q=$q NB=$w $(echo $r | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms"], d["split_ms"])' 2>/dev/null)"
done; done
