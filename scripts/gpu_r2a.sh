#!/bin/bash
# round-2 status check on the GPU box: tests, timings, bench
make -C paper_2508_04711_b200/csrc -j8 > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest.log
timeout 300 python scripts/time_c2.py > gpurun_out/time_c2.log 2>&1; echo "time rc=$?"; cat gpurun_out/time_c2.log | tail -10
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench.log
