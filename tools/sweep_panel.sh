#!/bin/bash
# time the n=4096 factorization for several panel CTA granularities
for mr in 8 16 28 48 64 128; do
  SKL_PANEL_MIN_ROWS=$mr python tools/run_blk.py --reps 2 | sed "s/^/min_rows=$mr /"
done
