#!/bin/bash
# build + plain bench (args forwarded) -> gpurun_out/bench.log
make -C paper_2508_04711_b200/csrc -j8 > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py "$@" > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log
