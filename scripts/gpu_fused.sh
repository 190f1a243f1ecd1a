#!/bin/bash
# fused backward bring-up on the GPU box
make -C paper_2508_04711_b200/csrc -j8 > gpurun_out/build_fused.log 2>&1 || { tail -20 gpurun_out/build_fused.log; exit 1; }
for w in small ragged mid c2; do
  echo "=== $w"
  timeout 120 python scripts/check_fused.py $w 2>&1 | tail -16
done
