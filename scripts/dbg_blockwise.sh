#!/bin/bash
# usage: scripts/dbg_blockwise.sh  (on the GPU box)
export CUDA_LAUNCH_BLOCKING=1
for a in "300 128 1.0" "300 128 0.5" "40 128 0.5" "40 64 0.5" "300,77,513 128 0.33" "3,2 64 0.5" "130 64 0.7"; do
  set -- $a
  echo "== $a"
  timeout 60 python scripts/dbg_blockwise.py $1 $2 $3 2>&1 | tail -3
  JH_DBG=4 timeout 60 python scripts/dbg_blockwise.py $1 $2 $3 2>&1 | tail -1
done
