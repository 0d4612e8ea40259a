#!/bin/bash
for d in 0 3 16 28 31; do
  SKL_PANEL_DBG=$d timeout 60 python tools/run_blk.py --reps 1 2>&1 | grep -E "ms|Error" | sed "s/^/dbg=$d /"
done
