# ncu evidence for profiles/: launch list of the bench command, and one --set full
# capture per attention kernel (each only after the plain bench exited 0).
mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-max-len > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_all.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-max-len > /dev/null 2>&1; echo launches=$?
for k in hstu_bwd_dkv hstu_fwd hstu_bwd_dq; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 -c 1 \
    -o gpurun_out/full_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-max-len > gpurun_out/full_$k.log 2>&1
  echo $k=$?
done
