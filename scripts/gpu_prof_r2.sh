#!/bin/bash
# round-2 ncu evidence: plain bench first, then the launch list and one --set full capture per attention kernel
make -C paper_2508_04711_b200/csrc -j8 > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
B="python bench.py --no-cpu-baseline --no-max-len --no-stack --no-e2e --cp-sweep-gb 0"
timeout 300 $B --steps 5 --warmup 3 > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err || { tail gpurun_out/prof_bench.err; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv \
  $B --steps 3 --warmup 3 > /dev/null 2>&1; echo launches=$?
for k in ${KERNELS:-hstu_bwd_dkv_kernel hstu_fwd_kernel hstu_bwd_dq_kernel}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 -c 1 \
    -o gpurun_out/full_$k -f $B --steps 1 --warmup 3 > gpurun_out/full_$k.log 2>&1
  echo $k=$?
done
