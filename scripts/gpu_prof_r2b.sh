#!/bin/bash
# round-2 extra evidence: helper bandwidths, fused-backward capture at long L, compute-sanitizer on smoke shapes
make -C paper_2508_04711_b200/csrc -j8 > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python scripts/bench_helpers.py gpurun_out/r2_helpers.json > gpurun_out/helpers.log 2>&1; echo helpers=$?; cat gpurun_out/helpers.log | tail -12
timeout 600 python scripts/fused_long.py > gpurun_out/fused_long.log 2>&1; echo fused_long=$?; tail -4 gpurun_out/fused_long.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hstu_bwd_fused_kernel -c 1 \
   -o gpurun_out/full_hstu_bwd_fused_kernel -f python scripts/fused_long.py --once > gpurun_out/full_fused.log 2>&1; echo ncu_fused=$?
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_smoke.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "$tool=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
