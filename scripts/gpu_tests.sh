#!/bin/bash
# build + the -m gpu suite (optionally a subset: scripts/gpu_tests.sh tests/test_x.py)
make -C paper_2508_04711_b200/csrc -j8 > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest ${@:-tests} -m gpu -x -q -s > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|error|Error|stack out|grad " gpurun_out/gputest.log | tail -40
