#!/bin/bash
# round-2: tests, fwd A/B, bench, launch list
make -C paper_2508_04711_b200/csrc -j8 > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest.log
JH_FWD1=1 timeout 300 python scripts/time_c2.py > gpurun_out/time_c2_fwd1.log 2>&1; echo "fwd1 rc=$?"; head -3 gpurun_out/time_c2_fwd1.log
timeout 300 python scripts/time_c2.py > gpurun_out/time_c2.log 2>&1; echo "time rc=$?"; head -3 gpurun_out/time_c2.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-max-len > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
