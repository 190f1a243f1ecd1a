# one full ncu capture of the dK/dV kernel (after a plain bench run exits 0)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-max-len > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K:-hstu_bwd_dkv} --launch-skip 3 -c 1 \
  -o gpurun_out/full_${K:-hstu_bwd_dkv} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-max-len > gpurun_out/ncu_one.log 2>&1
echo ncu=$?
